"""Lifetime order as a window staircase (csrc/fw2v_stair.cuh) vs the
one-window wavefront (k1s_snapshot<..., LIFETIME = true>, FW2V_NO_STAIR=1).

Both run the reference's sweep_samples order (trainer.cpp:133-154) with the
same FP operations per pairing, so on launches whose sentences cannot interact
(disjoint id ranges for rows and negatives) the two kernels must agree bit for
bit — including sentences of unequal length sharing a warp, windows with
repeated sample ids (serial fallback) and ids shared between consecutive
windows (tail finished before the window starts). Against the oracle the
staircase is covered by tests/test_parity_bench.py (lifetime, bench knobs).
"""
import os

import numpy as np
import pytest

from helpers import sgns_loss

pytestmark = pytest.mark.gpu
fw = pytest.importorskip("paper_2312_07743_b200")


def _run(stair, cfg, counts, inp, out, launches):
    old = os.environ.pop("FW2V_NO_STAIR", None)
    if not stair:
        os.environ["FW2V_NO_STAIR"] = "1"
    try:
        with fw.Trainer(cfg, counts) as t:
            t.set_model(inp, out)
            ctrs = []
            for offsets, ids, negs, alphas in launches:
                ctrs.append(t.train_sentences(offsets, ids, negs, alphas, serial=False).as_tuple())
            gi, go = t.get_model()
    finally:
        os.environ.pop("FW2V_NO_STAIR", None)
        if old is not None:
            os.environ["FW2V_NO_STAIR"] = old
    return gi, go, ctrs


def _disjoint_launch(rng, n_sent, band, lens, n_neg, types_per_band):
    """n_sent sentences, sentence s drawing ids and negatives only from band s
    (ids s*band .. s*band + types_per_band - 1): no row is shared between sentences."""
    ids, negs, offs = [], [], [0]
    for s in range(n_sent):
        L = int(lens[s])
        lo = s * band
        ids.append(rng.integers(lo, lo + types_per_band, L))
        negs.append(rng.integers(lo, lo + types_per_band, L * n_neg))
        offs.append(offs[-1] + L)
    alphas = rng.uniform(0.005, 0.05, n_sent).astype(np.float32)
    return (np.array(offs, np.uint64), np.concatenate(ids).astype(np.int32),
            np.concatenate(negs).astype(np.int32), alphas)


@pytest.mark.parametrize("dim", [64, 128, 256, 300])
@pytest.mark.parametrize("window", [2, 4, 5, 6, 8, 10])
@pytest.mark.parametrize("types_per_band", [7, 40, 500], ids=["repeats", "some", "rare"])
def test_stair_equals_wavefront_bitwise(dim, window, types_per_band):
    n_neg = 5
    rng = np.random.default_rng(dim * 100 + window * 10 + types_per_band)
    n_sent, band = 24, 600
    V = n_sent * band
    counts = (10 + V - np.arange(V)).astype(np.uint64)
    launches = []
    for _ in range(3):
        lens = rng.integers(1, 90, n_sent)
        lens[:4] = [1, 2, 3, 2 * window + 3][:4]  # edge lengths share warps with long sentences
        launches.append(_disjoint_launch(rng, n_sent, band, lens, n_neg, types_per_band))
    inp = ((rng.random((V, dim)) - 0.5) / dim).astype(np.float32)
    out = ((rng.random((V, dim)) - 0.5) * 0.5).astype(np.float32)
    cfg = fw.TrainConfig(dim=dim, window=window, negatives=n_neg, workers=4, deterministic=0,
                         reuse_mode="lifetime", fast_sigmoid=True, delta_writeback=2, l1_refresh_log2=0,
                         hot_rows=0)
    a_in, a_out, a_ctr = _run(True, cfg, counts, inp, out, launches)
    b_in, b_out, b_ctr = _run(False, cfg, counts, inp, out, launches)
    assert a_ctr == b_ctr
    assert np.isfinite(a_in).all() and np.isfinite(a_out).all()
    assert not np.array_equal(a_out, out), "nothing trained"
    assert np.array_equal(a_in, b_in), np.abs(a_in - b_in).max()
    assert np.array_equal(a_out, b_out), np.abs(a_out - b_out).max()


@pytest.mark.parametrize("hot_rows", [0, 64])
def test_stair_hogwild_text8_loss(ref, hot_rows):
    """One Hogwild epoch on the text8 shape: the staircase and the one-window
    wavefront (which differ only in Hogwild interleaving) each reach the reference
    train()'s SGNS loss within 2%. (On a 4,000-sentence subset the reference's own
    loss varied by 1.5% between runs of its 16 Hogwild threads; the whole corpus
    keeps that spread well below the tolerance.)"""
    from oracle.oracle import TrainConfig as RConfig

    corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
    base = dict(dim=128, window=5, negatives=5, epochs=1, batch_sentences=10000, subsample=1e-4, seed=3)
    p = corpus.counts.astype(np.float64) ** 0.75
    off = corpus.offsets[:2001].copy()
    negs = np.random.default_rng(5).choice(len(corpus.counts), int(off[-1]) * 5, p=p / p.sum()).astype(np.int32)

    def loss(i, o):
        return sgns_loss(i, o, off, corpus.ids[: int(off[-1])], negs, 3, 5, max_pairs=200_000)

    rin, rout, _ = ref.train(corpus.counts, corpus.offsets, corpus.ids, RConfig(workers=os.cpu_count() or 8, **base))
    ref_loss = loss(rin, rout)
    cfg = fw.TrainConfig(workers=64, streams=16, deterministic=0, reuse_mode="lifetime", sampler="alias",
                         hot_rows=hot_rows, **base)
    got = []
    for stair in (True, False):
        old = os.environ.pop("FW2V_NO_STAIR", None)
        if not stair:
            os.environ["FW2V_NO_STAIR"] = "1"
        try:
            with fw.Trainer(cfg, corpus.counts) as t:
                t.train_corpus(corpus)
                gi, go = t.get_model()
        finally:
            os.environ.pop("FW2V_NO_STAIR", None)
            if old is not None:
                os.environ["FW2V_NO_STAIR"] = old
        got.append(loss(gi, go))
    print(f"hot_rows={hot_rows}: loss stair {got[0]:.4f} wavefront {got[1]:.4f} reference {ref_loss:.4f}")
    for g in got:
        assert abs(g - ref_loss) / ref_loss <= 0.02


@pytest.mark.parametrize("types", [40, 2000], ids=["repeats", "rare"])
def test_stair_n15_per_sentence_vs_oracle(oracle, types):
    """N = 15 in lifetime order: the 16 samples stream through 2W_f register
    slots of the staircase (32-lane groups, 32 x 4 at d=128). One sentence per
    launch against the oracle's reference order (trainer.cpp:133-154), fast
    sigmoid: relative update error <= 1e-4 (repeated ids inside a window take the
    serial path with the row handed over, as the reference re-reads it)."""
    from oracle.oracle import TrainConfig as OConfig

    dim, n_neg, L, n = 128, 15, 120, 6
    rng = np.random.default_rng(types)
    V = max(types, 64)
    counts = (10 + V - np.arange(V)).astype(np.uint64)
    ids = rng.integers(0, types, n * L).astype(np.int32)
    offsets = (np.arange(n + 1) * L).astype(np.uint64)
    negs = rng.integers(0, types, n * L * n_neg).astype(np.int32)
    alphas = np.full(n, 0.025, np.float32)
    cfg = dict(dim=dim, window=5, negatives=n_neg, workers=4, reuse_mode="lifetime")
    ri = ((rng.random((V, dim)) - 0.5) / dim).astype(np.float32)
    ro = ((rng.random((V, dim)) - 0.5) * 0.5).astype(np.float32)
    gi0, go0 = ri.copy(), ro.copy()
    for s in range(n):
        o = offsets[s:s + 2] - offsets[s]
        oracle.train_sentences(ri, ro, o, ids[s * L:(s + 1) * L], negs[s * L * n_neg:(s + 1) * L * n_neg],
                               alphas[s:s + 1], OConfig(**cfg))
    with fw.Trainer(fw.TrainConfig(deterministic=0, hot_rows=0, fast_sigmoid=True, delta_writeback=2,
                                   l1_refresh_log2=0, **cfg), counts) as t:
        t.set_model(gi0, go0)
        for s in range(n):
            o = offsets[s:s + 2] - offsets[s]
            t.train_sentences(o, ids[s * L:(s + 1) * L], negs[s * L * n_neg:(s + 1) * L * n_neg], alphas[s:s + 1],
                              serial=False)
        gi, go = t.get_model()
    ei = np.linalg.norm((gi - ri).astype(np.float64)) / np.linalg.norm((ri - gi0).astype(np.float64))
    eo = np.linalg.norm((go - ro).astype(np.float64)) / np.linalg.norm((ro - go0).astype(np.float64))
    print(f"N=15 lifetime {types} types: relative update error input {ei:.2e} output {eo:.2e}")
    assert ei <= 1e-4 and eo <= 1e-4
