"""Embedding output writer: fw2v_write_embeddings must produce
the reference save_embeddings file (model.cpp:47-74) byte for byte, on any
number of threads. The reference writer is called through oracle/_ref."""
import numpy as np
import pytest

fw = pytest.importorskip("paper_2312_07743_b200")


def _names(n):
    return [f"w{i:09d}" for i in range(n)]  # ref_capi token names


def _rows(n, d, seed):
    rng = np.random.default_rng(seed)
    r = (rng.standard_normal((n, d)) * rng.choice([1e-8, 1e-3, 0.5, 3.0, 1e4], (n, 1))).astype(np.float32)
    # values that sit on or next to a 6-decimal rounding boundary, signed zeros, large and tiny magnitudes
    special = np.array([0.0, -0.0, 0.0078125, -0.0078125, 1e-7, -1e-7, 0.0000005, 0.9999995, 123456.789, -2.5e-6,
                        np.float32(1) / 3, 65504.0, 1e-30, -1e30], np.float32)
    k = min(len(special), r.size)
    r.ravel()[:k] = special[:k]
    return r


@pytest.mark.parametrize("n,d,threads", [(1, 1, 1), (7, 3, 1), (3000, 16, 4), (2500, 128, 0), (1100, 300, 16)])
def test_write_embeddings_matches_reference(ref, tmp_path, n, d, threads):
    rows = _rows(n, d, seed=n + d)
    counts = (10 * n + 100 - np.arange(n)).astype(np.uint64)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    fw.fw2v.write_embeddings(ours, rows, _names(n), threads=threads)
    ref.save_embeddings(theirs, rows, counts)
    assert ours.read_bytes() == theirs.read_bytes()


def test_write_embeddings_errors(tmp_path):
    rows = np.zeros((2, 4), np.float32)
    with pytest.raises(fw.fw2v.Fw2vError) as e:
        fw.fw2v.write_embeddings(tmp_path / "no" / "such" / "dir.txt", rows, ["a", "b"])
    assert e.value.code == 1  # ringvec ErrorCode::io + 1
    with pytest.raises(ValueError):
        fw.fw2v.write_embeddings(tmp_path / "x.txt", rows, ["a"])


@pytest.mark.gpu
def test_save_model_from_device_matches_reference(ref, tmp_path):
    """Trainer.save_model (device -> host -> parallel text) == reference
    save_embeddings of the same matrices (padded rows at d=100 included)."""
    n, d = 3000, 100
    counts = (10 * n + 100 - np.arange(n)).astype(np.uint64)
    inp, out = _rows(n, d, 1), _rows(n, d, 2)
    with fw.Trainer(fw.TrainConfig(dim=d, workers=4), counts) as t:
        t.set_model(inp, out)
        for which, m in (("input", inp), ("output", out)):
            ours, theirs = tmp_path / f"ours_{which}.txt", tmp_path / f"ref_{which}.txt"
            t.save_model(ours, _names(n), which=which)
            ref.save_embeddings(theirs, m, counts)
            assert ours.read_bytes() == theirs.read_bytes()


def test_write_embeddings_bit_patterns_match_reference(ref, tmp_path):
    """Random float bit patterns over the whole exponent range (subnormals,
    rounding ties, huge values, inf, nan) against the reference writer."""
    rng = np.random.default_rng(11)
    n, d = 2000, 100
    bits = rng.integers(0, 2**32, n * d, dtype=np.uint64).astype(np.uint32)
    rows = bits.view(np.float32).reshape(n, d).copy()
    # plus every exponent with a few mantissas near .5 ulp-of-1e-6 boundaries
    e = np.arange(0, 255, dtype=np.uint32)
    rows.ravel()[: 255] = ((e << 23) | 0x400000).view(np.float32)
    counts = (10 * n + 100 - np.arange(n)).astype(np.uint64)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    fw.fw2v.write_embeddings(ours, rows, _names(n), threads=3)
    ref.save_embeddings(theirs, rows, counts)
    assert ours.read_bytes() == theirs.read_bytes()
