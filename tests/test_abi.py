"""C-ABI checks that need no GPU: libfw2v.so loads, exports every symbol
include/fw2v.h declares, its host batcher primitives equal the oracle, and the
training entry points fail loudly (no CPU fallback) when no device exists."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2312_07743_b200 as fw
from helpers import random_corpus

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "fw2v.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fw2v_[a-z0-9_]+)\s*\(", text)) - {"fw2v_observer_fn", "fw2v_epoch_fn"})


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(fw.fw2v.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(fw.fw2v.EXPORTED) == syms
    assert lib.fw2v_abi_version() == 1


def test_dropin_library_present():
    assert os.path.exists(fw.fw2v.DROPIN_PATH)


def test_config_defaults_mirror_trainconfig(oracle):
    c = fw.fw2v.CConfig()
    fw.fw2v.lib().fw2v_config_default(ctypes.byref(c))
    ref = fw.TrainConfig()
    for name in ["dim", "window", "negatives", "epochs", "min_count", "batch_sentences", "max_sentence_len",
                 "workers", "seed", "table_size", "queue_capacity"]:
        assert getattr(c, name) == getattr(ref, name), name
    assert c.alpha0 == pytest.approx(0.025) and c.subsample == 1e-4 and c.table_power == 0.75


def test_extension_defaults_mirror_python():
    """The C defaults of the B200 extension fields equal the Python dataclass's
    (TrainConfig.to_c writes every field, so the two must not drift)."""
    c = fw.fw2v.CConfig()
    fw.fw2v.lib().fw2v_config_default(ctypes.byref(c))
    py = fw.TrainConfig().to_c()
    for name, _ in fw.fw2v.CConfig._fields_:
        if name in ("workers",):
            continue
        assert getattr(c, name) == getattr(py, name), name
    assert c.divergence_guard == 1


def test_validate_config_rejects_like_reference():
    bad = fw.fw2v.CConfig()
    fw.fw2v.lib().fw2v_config_default(ctypes.byref(bad))
    assert fw.fw2v.lib().fw2v_validate_config(ctypes.byref(bad)) == 0
    for field, val in [("dim", 0), ("window", 0), ("negatives", -1), ("epochs", -1), ("alpha0", 0.0),
                       ("batch_sentences", 0), ("table_size", 0), ("min_count", 0)]:
        c = fw.fw2v.CConfig()
        fw.fw2v.lib().fw2v_config_default(ctypes.byref(c))
        setattr(c, field, val)
        assert fw.fw2v.lib().fw2v_validate_config(ctypes.byref(c)) == fw.fw2v.ERR_BAD_CONFIG, field


@pytest.mark.parametrize("threshold", [0.0, 1e-4, 1e-2])
def test_keep_probs_equal_oracle(oracle, threshold):
    counts = np.sort(np.random.default_rng(1).integers(1, 10**6, 500))[::-1].astype(np.uint64)
    a, b = fw.keep_probs(counts, threshold), oracle.keep_probs(counts, threshold)
    if threshold <= 0:
        assert a is None and b is None
    else:
        np.testing.assert_array_equal(a, b)


def test_table_equals_oracle(oracle):
    counts = np.sort(np.random.default_rng(2).integers(1, 10**5, 300))[::-1].astype(np.uint64)
    np.testing.assert_array_equal(fw.table(counts, 0.75, 100_003), oracle.table(counts, 0.75, 100_003))


@pytest.mark.parametrize("sub,n_neg", [(1e-2, 5), (0.0, 3), (1e-3, 0)])
def test_assemble_batch_equals_oracle(oracle, sub, n_neg):
    counts, offsets, ids = random_corpus(60, 40, 80, 3)
    cursor = 0
    k = 0
    while cursor < len(offsets) - 1:
        x = fw.assemble_batch(counts, offsets, ids, cursor, 9, n_neg, 0.75, 5003, sub, 11, 0, 0, k)
        y = oracle.assemble_batch(counts, offsets, ids, cursor, 9, n_neg, 0.75, 5003, sub, 11, 0, 0, k)
        assert x[0] == y[0]
        for p, q in zip(x[1:], y[1:]):
            np.testing.assert_array_equal(p, q)
        cursor = x[0]
        k += 1


def test_lr_and_analytic_equal_oracle(oracle):
    for w, t in [(0, 10), (3, 10), (10, 10), (11, 10), (123456, 1000000)]:
        assert fw.lr_at(w, t, 0.025) == oracle.lr_at(w, t, 0.025)
    for length in [1, 2, 3, 7, 30]:
        for width in [1, 3, 4]:
            for mode in ["lifetime", "window", "none", "window_snapshot"]:
                assert fw.analytic_traffic(length, width, 5, mode) == oracle.analytic_traffic(length, width, 5, mode)


def test_synth_zipf_shape_and_determinism():
    a = fw.synth_zipf(types=5000, tokens=200_000, sentence_len=1000)
    b = fw.synth_zipf(types=5000, tokens=200_000, sentence_len=1000, threads=3)
    np.testing.assert_array_equal(a.counts, b.counts)
    np.testing.assert_array_equal(a.offsets, b.offsets)
    np.testing.assert_array_equal(a.ids, b.ids)
    assert (np.diff(a.counts.astype(np.int64)) <= 0).all()  # count-descending vocabulary
    assert a.counts.min() >= 5 and a.ids.max() < len(a.counts)
    assert int(a.counts.sum()) == len(a.ids)
    assert (np.diff(a.offsets) <= 1000).all() and a.n_sentences == 200


def test_text8_shape_matches_baseline():
    c = fw.synth_zipf(**fw.TEXT8_SHAPE)
    assert c.n_sentences == 16_719
    assert abs(len(c.counts) - 71_290) <= 5  # ~71,290 types survive min_count 5


@pytest.mark.skipif(fw.device_count() > 0, reason="a CUDA device is present")
def test_training_fails_loudly_without_device():
    counts = np.arange(100, 0, -1).astype(np.uint64)
    with pytest.raises(fw.Fw2vError) as e:
        fw.Trainer(fw.TrainConfig(dim=16), counts)
    assert e.value.code == fw.fw2v.ERR_NO_DEVICE


def test_alias_sampler_vector_and_scalar_paths_agree():
    """The AVX-512 batching kernels (alias draws, subsampling) produce exactly
    the scalar sequence: the same draws from the run with FW2V_NO_AVX512 set."""
    import os
    import subprocess
    import sys

    code = ("import numpy as np, paper_2312_07743_b200 as fw;"
            "c=(np.arange(5000,0,-1)**1.5).astype(np.uint64);"
            "print(fw.fw2v.alias_draws(c,0.75,7,100003).astype(np.int64).tobytes().hex())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"FW2V_NO_AVX512": "1"}):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root,
                           env={**os.environ, **env}, check=True)
        outs.append(r.stdout.strip())
    assert outs[0] == outs[1]


def test_alias_sampler_distribution():
    """Draw frequencies follow count^0.75 (chi-square over the top 200 words)."""
    import numpy as np

    c = (np.arange(5000, 0, -1) ** 1.5).astype(np.uint64)
    d = fw.fw2v.alias_draws(c, 0.75, 3, 2_000_000)
    p = c.astype(np.float64) ** 0.75
    p /= p.sum()
    obs = np.bincount(d, minlength=len(c))[:200]
    exp = p[:200] * len(d)
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert chi2 < 300  # 199 dof: mean 199, sd ~20
