"""GPU evaluation scans vs the reference eval.cpp: identical
neighbours (ids, order and cosine values) and identical analogy predictions.
Embeddings include duplicate rows (exact ties, broken by id) and zero rows
(skipped as untrained)."""
import numpy as np
import pytest

fw = pytest.importorskip("paper_2312_07743_b200")


def _emb(n, d, seed):
    rng = np.random.default_rng(seed)
    rows = rng.standard_normal((n, d)).astype(np.float32)
    rows[5] = rows[3]          # exact tie for every query
    rows[17] = 2.0 * rows[11]  # same direction, different norm
    rows[7] = 0.0              # untrained row
    return rows


def test_eval_no_device_is_an_error():
    if fw.device_count() > 0:
        pytest.skip("has a device")
    with pytest.raises(fw.fw2v.Fw2vError) as e:
        fw.fw2v.nearest_neighbors(_emb(50, 8, 0), [1, 2], 5)
    assert e.value.code == 66


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,k", [(50, 8, 5), (3000, 128, 10), (2000, 300, 32), (20000, 64, 10)])
def test_nearest_neighbors_match_reference(ref, n, d, k):
    rows = _emb(n, d, seed=n + d)
    queries = np.array([0, 3, 5, 11, 17, n - 1] + list(range(20, min(n, 60))), np.int32)
    gi, gc = fw.fw2v.nearest_neighbors(rows, queries, k)
    ri, rc = ref.nearest_neighbors(rows, queries, k)
    np.testing.assert_array_equal(gi, ri)
    np.testing.assert_array_equal(gc, rc)


@pytest.mark.gpu
def test_nearest_neighbors_errors():
    rows = _emb(50, 8, 1)
    for args, code in (((rows, [1], 0), 4), ((rows, [1], 50), 4), ((rows, [50], 5), 11), ((rows, [7], 5), 12)):
        with pytest.raises(fw.fw2v.Fw2vError) as e:
            fw.fw2v.nearest_neighbors(*args)
        assert e.value.code == code


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["cos_add", "cos_mul"])
@pytest.mark.parametrize("n,d", [(60, 8), (5000, 128), (3000, 300)])
def test_analogy_predictions_match_reference(ref, method, n, d):
    rows = _emb(n, d, seed=7 * n + d)
    rng = np.random.default_rng(n)
    quads = rng.integers(0, n, (200, 3)).astype(np.int32)
    quads[:5] = [[3, 11, 17], [5, 3, 11], [11, 17, 3], [0, 7, 1], [2, 2, 4]]  # ties, zero row, repeats
    pred, acc = fw.fw2v.eval_analogy(rows, np.concatenate([quads, np.zeros((len(quads), 1), np.int32)], 1), method)
    full = np.concatenate([quads, pred[:, None]], 1)
    ok = ref.analogy_correct(rows, full, 0 if method == "cos_add" else 1)
    assert ok.all(), np.nonzero(ok == 0)[0][:10]
    _, acc2 = fw.fw2v.eval_analogy(rows, full, method)
    assert acc2 == 1.0
