"""GPU parity: the B200 kernels through the C-ABI vs the CPU oracle.

Tier 1 (deterministic): the serial exact engine K2 must equal
the oracle (and so the reference built with default flags) bit for bit.
Tier 2 (Hogwild K1): per-sentence semantics equal the reference up to float
association (checked with one sentence in flight), counters equal the closed
forms, and full Hogwild runs stay within the loss tolerance.
"""
import numpy as np
import pytest

from helpers import distinct_corpus, fixed_negatives, random_corpus

pytestmark = pytest.mark.gpu

fw = pytest.importorskip("paper_2312_07743_b200")
from oracle.oracle import TrainConfig as OConfig  # noqa: E402


def _trainer(**kw):
    counts = kw.pop("counts")
    return fw.Trainer(fw.TrainConfig(**kw), counts)


@pytest.mark.parametrize("dim", [4, 8, 12, 16, 24, 32, 100, 128, 300])
def test_init_model_bitwise(oracle, dim):
    V = 37
    counts = (1000 - np.arange(V)).astype(np.uint64)
    with _trainer(counts=counts, dim=dim, seed=123, workers=1) as t:
        gi, go = t.get_model()
    ri, ro = oracle.init_model(V, dim, 123)
    assert np.array_equal(gi, ri)
    assert not go.any()


@pytest.mark.parametrize("mode", ["lifetime", "window", "none", "window_snapshot"])
@pytest.mark.parametrize("dim,window,n_neg", [(8, 5, 5), (12, 7, 3), (16, 2, 0), (32, 5, 5), (128, 5, 5), (300, 5, 5)])
def test_k2_train_sentences_bitwise(oracle, mode, dim, window, n_neg):
    counts, offsets, ids = random_corpus(12, 20, 15, seed=dim + window)  # small vocab: collisions
    V = len(counts)
    negs = fixed_negatives(int(offsets[-1]), n_neg, V, seed=3)
    alphas = np.linspace(0.025, 0.01, len(offsets) - 1).astype(np.float32)
    cfg = dict(dim=dim, window=window, negatives=n_neg, reuse_mode=mode, workers=1)
    ri, ro = oracle.init_model(V, dim, 5)
    ro = (ri[::-1] * 0.5).copy()  # non-zero output so every pairing moves
    ri0, ro0 = ri.copy(), ro.copy()
    rc = oracle.train_sentences(ri, ro, offsets, ids, negs, alphas, OConfig(**cfg))
    with _trainer(counts=counts, **cfg) as t:
        t.set_model(ri0, ro0)
        c = t.train_sentences(offsets, ids, negs, alphas, serial=True)
        gi, go = t.get_model()
    assert c.as_tuple() == rc
    np.testing.assert_array_equal(gi, ri)
    np.testing.assert_array_equal(go, ro)


@pytest.mark.parametrize("dim,window,n_neg,sub", [(12, 5, 5, 1e-2), (16, 7, 3, 0.0), (128, 5, 5, 1e-3)])
def test_train_deterministic_bitwise(oracle, dim, window, n_neg, sub):
    counts, offsets, ids = random_corpus(60, 30, 40, seed=dim)
    cfg = dict(dim=dim, window=window, negatives=n_neg, epochs=2, workers=1, batch_sentences=7,
               table_size=5003, subsample=sub, seed=42)
    ri, ro, rrep = oracle.train(counts, offsets, ids, OConfig(**cfg))
    with _trainer(counts=counts, **cfg) as t:
        rep = t.train_corpus(fw.Corpus(counts, offsets, ids))
        gi, go = t.get_model()
    assert rep.words_trained == rrep.words_trained
    assert rep.traffic == rrep.traffic == rrep.analytic
    assert [e["words"] for e in rep.epochs] == rrep.epoch_words
    np.testing.assert_array_equal(gi, ri)
    np.testing.assert_array_equal(go, ro)


@pytest.mark.parametrize("dim,lanes", [(8, 0), (12, 0), (16, 0), (32, 0), (64, 0), (128, 0), (128, 32), (128, 16),
                                       (128, 8), (256, 0), (300, 0), (512, 0)])
@pytest.mark.parametrize("window", [2, 5, 7])
@pytest.mark.parametrize("mode", ["lifetime", "window_snapshot"])
def test_k1_single_sentence_semantics(oracle, dim, lanes, window, mode):
    """K1 with one sentence per launch == reference order up to FP association
    (precise sigmoid); duplicates and negative collisions included."""
    counts, offsets, ids = random_corpus(6, 40, 25, seed=dim * 7 + window, min_len=1)
    V = len(counts)
    n_neg = 5
    negs = fixed_negatives(int(offsets[-1]), n_neg, V, seed=9)
    alphas = np.full(len(offsets) - 1, 0.025, np.float32)
    cfg = dict(dim=dim, window=window, negatives=n_neg, workers=4, reuse_mode=mode)
    gcfg = dict(cfg, deterministic=0, fast_sigmoid=False, k1_lanes=lanes, l1_refresh_log2=0, delta_writeback=False,
                hot_rows=0)
    ri, _ = oracle.init_model(V, dim, 5)
    ro = (ri[::-1] * 4.0).copy()
    gi0, go0 = ri.copy(), ro.copy()
    rc_total = np.zeros(5, np.uint64)
    for s in range(len(offsets) - 1):
        o = offsets[s:s + 2] - offsets[s]
        sl = ids[int(offsets[s]):int(offsets[s + 1])]
        ng = negs[int(offsets[s]) * n_neg:int(offsets[s + 1]) * n_neg]
        rc_total += np.array(oracle.train_sentences(ri, ro, o, sl, ng, alphas[s:s + 1], OConfig(**cfg)), np.uint64)
    with _trainer(counts=counts, **gcfg) as t:
        t.set_model(gi0, go0)
        tot = np.zeros(5, np.uint64)
        for s in range(len(offsets) - 1):
            o = offsets[s:s + 2] - offsets[s]
            sl = ids[int(offsets[s]):int(offsets[s + 1])]
            ng = negs[int(offsets[s]) * n_neg:int(offsets[s + 1]) * n_neg]
            tot += np.array(t.train_sentences(o, sl, ng, alphas[s:s + 1], serial=False).as_tuple(), np.uint64)
        gi, go = t.get_model()
    assert tuple(tot) == tuple(rc_total)
    scale_i = np.abs(ri).max()
    scale_o = np.abs(ro).max()
    assert np.abs(gi - ri).max() <= 2e-5 * scale_i + 1e-7
    assert np.abs(go - ro).max() <= 2e-5 * scale_o + 1e-7


def test_k1_distinct_tokens_batch_equals_serial(oracle):
    """Sentences with globally disjoint rows do not interact, so a whole Hogwild
    batch equals serial training up to FP association."""
    n, L = 64, 30
    rng = np.random.default_rng(1)
    types = n * L + 10
    ids = rng.permutation(types)[: n * L].astype(np.int32)
    offsets = (np.arange(n + 1) * L).astype(np.uint64)
    counts = (100 + types - np.arange(types)).astype(np.uint64)
    n_neg = 0  # negatives would share rows across sentences
    alphas = np.full(n, 0.025, np.float32)
    cfg = dict(dim=64, window=5, negatives=n_neg, workers=4)
    ri, _ = oracle.init_model(types, 64, 3)
    ro = (ri[::-1] * 4.0).copy()
    gi0, go0 = ri.copy(), ro.copy()
    oracle.train_sentences(ri, ro, offsets, ids, np.zeros(0, np.int32), alphas, OConfig(**cfg))
    with _trainer(counts=counts, deterministic=0, fast_sigmoid=False, hot_rows=0, **cfg) as t:
        t.set_model(gi0, go0)
        t.train_sentences(offsets, ids, np.zeros(0, np.int32), alphas, serial=False)
        gi, go = t.get_model()
    assert np.abs(gi - ri).max() <= 1e-6
    assert np.abs(go - ro).max() <= 1e-5


def test_hogwild_counters_and_words():
    counts, offsets, ids = random_corpus(300, 40, 200, seed=4)
    cfg = dict(dim=32, window=5, negatives=5, epochs=2, workers=4, batch_sentences=16, table_size=10007,
               subsample=1e-2, seed=31, deterministic=0)
    with _trainer(counts=counts, **cfg) as t:
        rep = t.train_corpus(fw.Corpus(counts, offsets, ids))
        gi, go = t.get_model()
    assert rep.traffic == rep.analytic
    assert rep.traffic[0] == rep.words_trained
    assert sum(e["words"] for e in rep.epochs) == rep.words_trained
    assert np.isfinite(gi).all() and np.isfinite(go).all()


def test_hogwild_uses_reference_batches(ref):
    """With the reference sampler the Hogwild run trains exactly the batches the
    reference assembles for the same workers (same streams derive(seed,e,p,k))."""
    counts, offsets, ids = random_corpus(200, 40, 100, seed=8)
    cfg = dict(dim=16, window=5, negatives=5, epochs=1, workers=3, batch_sentences=11, table_size=10007,
               subsample=1e-2, seed=5)
    _, _, rrep = ref.train(counts, offsets, ids, OConfig(**cfg))
    with _trainer(counts=counts, deterministic=0, **cfg) as t:
        rep = t.train_corpus(fw.Corpus(counts, offsets, ids))
    assert rep.words_trained == rrep.words_trained
    assert rep.sentences_trained == rrep.sentences_trained
    assert rep.analytic == rrep.analytic


def _disjoint_batch(n, L, pool, n_neg, seed, distinct=False):
    """n sentences of length L whose ids and negatives come from disjoint
    per-sentence token pools: Hogwild sentences never share a row. distinct:
    no token repeats inside a sentence (pool >= L)."""
    rng = np.random.default_rng(seed)
    pick = (lambda k: rng.permutation(pool)[:k]) if distinct else (lambda k: rng.integers(0, pool, k))
    ids = np.concatenate([s * pool + pick(L) for s in range(n)]).astype(np.int32)
    negs = np.concatenate([s * pool + rng.integers(0, pool, L * n_neg) for s in range(n)]).astype(np.int32)
    offsets = (np.arange(n + 1) * L).astype(np.uint64)
    counts = (100 + n * pool - np.arange(n * pool)).astype(np.uint64)
    return counts, offsets, ids, negs


@pytest.mark.parametrize("dim", [16, 32, 64, 128, 256, 300, 512])
@pytest.mark.parametrize("delta", [False, True])
def test_k1s_disjoint_batch_equals_serial(oracle, dim, delta):
    """A whole Hogwild K1s batch (several sentences per warp at small lane
    counts) over row-disjoint sentences equals the reference snapshot order
    applied sentence by sentence, up to FP association. Overwrite write-back:
    duplicates inside a sentence included; delta write-back (red.add of the
    ring rows' final - loaded) is exact when a sentence's ring never holds one
    token twice."""
    n, L, n_neg = 96, 40, 5
    pool = 48 if delta else 12
    counts, offsets, ids, negs = _disjoint_batch(n, L, pool, n_neg, seed=dim, distinct=delta)
    V = len(counts)
    alphas = np.full(n, 0.025, np.float32)
    cfg = dict(dim=dim, window=5, negatives=n_neg, workers=4, reuse_mode="window_snapshot")
    ri, _ = oracle.init_model(V, dim, 3)
    ro = (ri[::-1] * 4.0).copy()
    gi0, go0 = ri.copy(), ro.copy()
    oracle.train_sentences(ri, ro, offsets, ids, negs, alphas, OConfig(**cfg))
    with _trainer(counts=counts, deterministic=0, fast_sigmoid=False, hot_rows=0, l1_refresh_log2=0,
                  delta_writeback=delta, **cfg) as t:
        t.set_model(gi0, go0)
        t.train_sentences(offsets, ids, negs, alphas, serial=False)
        gi, go = t.get_model()
    assert np.abs(gi - ri).max() <= 2e-5 * np.abs(ri).max() + 1e-7
    assert np.abs(go - ro).max() <= 2e-5 * np.abs(ro).max() + 1e-7


@pytest.mark.parametrize("replicas", [1, 2, 4])
@pytest.mark.parametrize("hot_merge", [0, 1], ids=["mean", "live"])
def test_k1s_hot_replicas_average(oracle, replicas, hot_merge):
    """Hot-row replicas: rows < hot_rows are trained by sentence s on replica
    s mod R. With one sentence its replica holds the reference update and the
    other R-1 replicas the untouched rows: the pass-end mean (hot_merge = 0)
    leaves hot output rows at v0 + (v_ref - v0) / R, the live merge (1) at the
    reference update itself; everything else is exact either way."""
    dim, n_neg, hot = 128, 5, 20
    counts, offsets, ids = random_corpus(1, 60, 40, seed=11, min_len=60)
    V = len(counts)
    negs = fixed_negatives(int(offsets[-1]), n_neg, V, seed=2)
    alphas = np.full(1, 0.025, np.float32)
    cfg = dict(dim=dim, window=5, negatives=n_neg, workers=4, reuse_mode="window_snapshot")
    ri, _ = oracle.init_model(V, dim, 5)
    ro = (ri[::-1] * 4.0).copy()
    gi0, go0 = ri.copy(), ro.copy()
    oracle.train_sentences(ri, ro, offsets, ids, negs, alphas, OConfig(**cfg))
    with _trainer(counts=counts, deterministic=0, fast_sigmoid=False, l1_refresh_log2=0, delta_writeback=False,
                  hot_rows=hot, hot_replicas=replicas, hot_merge=hot_merge, **cfg) as t:
        t.set_model(gi0, go0)
        t.train_sentences(offsets, ids, negs, alphas, serial=False)
        gi, go = t.get_model()
    want = ro.copy()
    if hot_merge == 0:
        want[:hot] = go0[:hot] + (ro[:hot] - go0[:hot]) / replicas
    assert np.abs(gi - ri).max() <= 2e-5 * np.abs(ri).max() + 1e-7
    assert np.abs(go - want).max() <= 2e-5 * np.abs(ro).max() + 1e-7


@pytest.mark.parametrize("dim", [32, 64, 128, 300, 512])
def test_k1s_overwrite_without_ring_matches_delta(dim):
    """delta_writeback=2 (ring rows stored straight back, no shared-memory ring;
    fast-sigmoid kernels) equals the delta write-back on row-disjoint sentences
    with distinct ring tokens, where neither can lose an update."""
    n, L, n_neg, pool = 96, 40, 5, 48
    counts, offsets, ids, negs = _disjoint_batch(n, L, pool, n_neg, seed=dim + 1, distinct=True)
    V = len(counts)
    alphas = np.full(n, 0.025, np.float32)
    rng = np.random.default_rng(dim)
    gi0 = ((rng.random((V, dim)) - 0.5) / dim).astype(np.float32)
    go0 = ((rng.random((V, dim)) - 0.5) / dim).astype(np.float32)
    out = {}
    for mode in (1, 2):
        with _trainer(counts=counts, dim=dim, window=5, negatives=n_neg, workers=4, reuse_mode="window_snapshot",
                      deterministic=0, fast_sigmoid=True, hot_rows=0, l1_refresh_log2=0, delta_writeback=mode) as t:
            t.set_model(gi0, go0)
            t.train_sentences(offsets, ids, negs, alphas, serial=False)
            out[mode] = t.get_model()
    for a, b in zip(out[1], out[2]):
        assert np.abs(a - b).max() <= 1e-6 * np.abs(a).max() + 1e-8


@pytest.mark.parametrize("mode", ["lifetime", "window_snapshot"])
@pytest.mark.parametrize("dim,window,n_neg", [(128, 5, 0), (128, 5, 2), (128, 5, 15), (32, 5, 15), (128, 9, 15),
                                              (64, 3, 9), (300, 5, 11), (512, 5, 5), (512, 3, 5), (512, 5, 15),
                                              (512, 9, 15), (512, 9, 5), (512, 1, 2), (128, 2, 15), (64, 3, 13),
                                              (256, 2, 12)])
def test_k1s_negative_counts_single_sentence(oracle, mode, dim, window, n_neg):
    """K1s with any number of negatives (partial chunk, several chunks per window;
    lifetime order: one wavefront per chunk) == the reference order per sentence,
    up to FP association; sentences with repeated ids included."""
    counts, offsets, ids = random_corpus(4, 40, 20, seed=dim + 3 * n_neg + window, min_len=1)
    V = len(counts)
    negs = fixed_negatives(int(offsets[-1]), n_neg, V, seed=n_neg)
    alphas = np.full(len(offsets) - 1, 0.025, np.float32)
    cfg = dict(dim=dim, window=window, negatives=n_neg, workers=4, reuse_mode=mode)
    gcfg = dict(cfg, deterministic=0, fast_sigmoid=False, l1_refresh_log2=0, delta_writeback=False, hot_rows=0)
    ri, _ = oracle.init_model(V, dim, 5)
    ro = (ri[::-1] * 4.0).copy()
    gi0, go0 = ri.copy(), ro.copy()
    for s in range(len(offsets) - 1):
        o = offsets[s:s + 2] - offsets[s]
        sl = ids[int(offsets[s]):int(offsets[s + 1])]
        ng = negs[int(offsets[s]) * n_neg:int(offsets[s + 1]) * n_neg]
        oracle.train_sentences(ri, ro, o, sl, ng, alphas[s:s + 1], OConfig(**cfg))
    with _trainer(counts=counts, **gcfg) as t:
        t.set_model(gi0, go0)
        for s in range(len(offsets) - 1):
            o = offsets[s:s + 2] - offsets[s]
            sl = ids[int(offsets[s]):int(offsets[s + 1])]
            ng = negs[int(offsets[s]) * n_neg:int(offsets[s + 1]) * n_neg]
            t.train_sentences(o, sl, ng, alphas[s:s + 1], serial=False)
        gi, go = t.get_model()
    assert np.abs(gi - ri).max() <= 2e-5 * np.abs(ri).max() + 1e-7
    assert np.abs(go - ro).max() <= 2e-5 * np.abs(ro).max() + 1e-7
