"""Parity pinned at the configurations the bench actually runs.

1. Tier 1 at the BASELINE text8 shape: the deterministic engine K2 trains one
   epoch of the text8-shaped corpus (16,719 sentences, 9.9 M trained words) at
   d=128 and d=300 and must equal the REFERENCE ringvec::train(workers=1)
   (trainer.cpp:390-528) bit for bit. The reference's matrices are pinned by
   SHA-256 in tests/golden/text8_ref_workers1.json (made by
   tests/golden/make_text8_golden.py from oracle/_ref, the reference compiled
   from its sources); the box has no /root/reference.
2. The K1s fast path with the bench's own knobs (tanh.approx sigmoid, L1-staged
   sample rows refreshed every 2^5 windows, ring-less overwrite write-back),
   one sentence per launch, against the oracle's per-sentence reference order
   with explicit tolerances on the relative update error.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
fw = pytest.importorskip("paper_2312_07743_b200")
from oracle.oracle import TrainConfig as OConfig  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "text8_ref_workers1.json")


def _digest(m):
    return hashlib.sha256(np.ascontiguousarray(m, dtype="<f4").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def text8():
    return fw.synth_zipf(**fw.TEXT8_SHAPE)


@pytest.mark.parametrize("dim", [128, 300])
def test_text8_k2_equals_reference(text8, dim):
    with open(GOLDEN) as f:
        g = json.load(f)
    h = hashlib.sha256()
    for a in (text8.counts, text8.offsets, text8.ids):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == g["corpus"]["sha256"], "synthetic text8 corpus differs from the golden run's"
    want = g["runs"][str(dim)]
    cfg = fw.TrainConfig(dim=dim, **g["config"])  # workers=1: serial exact engine K2
    with fw.Trainer(cfg, text8.counts) as t:
        rep = t.train_corpus(text8)
        gi, go = t.get_model()
    assert rep.words_trained == want["words_trained"]
    assert rep.sentences_trained == want["sentences_trained"]
    assert list(rep.traffic) == want["traffic"]
    info = (f"fro {np.linalg.norm(gi.astype(np.float64)):.9g}/{want['input_fro']:.9g} "
            f"{np.linalg.norm(go.astype(np.float64)):.9g}/{want['output_fro']:.9g} "
            f"row1 {gi[1, :4]} vs {want['input_row1_head'][:4]}")
    assert _digest(gi) == want["input_sha256"], info
    assert _digest(go) == want["output_sha256"], info


def _zipf_sentences(text8, n, length, seed):
    """n sentences of `length` post-subsampling-like ids drawn from the text8
    corpus (Zipf-hot rows repeat inside a sentence, as in the bench)."""
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, len(text8.ids) - length, n)
    ids = np.concatenate([text8.ids[s:s + length] for s in starts]).astype(np.int32)
    offsets = (np.arange(n + 1) * length).astype(np.uint64)
    return offsets, ids


def _unigram_negatives(counts, n, seed):
    p = counts.astype(np.float64) ** 0.75
    return np.random.default_rng(seed).choice(len(counts), n, p=p / p.sum()).astype(np.int32)


# (name, knobs, bound on ||gpu - ref|| / ||ref - init|| per matrix)
KNOBS = [
    ("fast_sigmoid", dict(fast_sigmoid=True, l1_refresh_log2=0, delta_writeback=0), 1e-4),
    ("fast+overwrite", dict(fast_sigmoid=True, l1_refresh_log2=0, delta_writeback=2), 1e-4),
    ("bench: fast+overwrite+l1_refresh5", dict(fast_sigmoid=True, l1_refresh_log2=5, delta_writeback=2), 1e-4),
]


@pytest.mark.parametrize("mode", ["window_snapshot", "lifetime"])
@pytest.mark.parametrize("dim", [128, 300])
@pytest.mark.parametrize("knobs", KNOBS, ids=[k[0] for k in KNOBS])
def test_k1s_bench_knobs_per_sentence(text8, oracle, mode, dim, knobs):
    """One sentence per launch (no Hogwild interaction): the bench kernel's
    deviations from the reference order are the fast sigmoid (|err| < 1e-3) and,
    with l1_refresh_log2 = 5, a sentence re-reading a sample row it rewrote
    within the last 32 windows from its SM's L1 — except that K1s re-reads a row
    the previous window rewrote, so inside one sentence the staging is exact.
    Measured (r02): relative update error <= 2e-6 for every knob set.)"""
    name, kn, bound = knobs
    n, L, n_neg = 6, 160, 5
    offsets, ids = _zipf_sentences(text8, n, L, seed=dim)
    V = len(text8.counts)
    negs = _unigram_negatives(text8.counts, n * L * n_neg, seed=dim + 1)
    alphas = np.full(n, 0.025, np.float32)
    cfg = dict(dim=dim, window=5, negatives=n_neg, workers=4, reuse_mode=mode)
    # A trained-looking start: small random rows in both matrices.
    rng = np.random.default_rng(dim)
    ri = ((rng.random((V, dim)) - 0.5) / dim).astype(np.float32)
    ro = ((rng.random((V, dim)) - 0.5) * 0.5).astype(np.float32)
    gi0, go0 = ri.copy(), ro.copy()
    from oracle.oracle import Oracle

    orc = Oracle("oracle")
    for s in range(n):
        o = offsets[s:s + 2] - offsets[s]
        orc.train_sentences(ri, ro, o, ids[s * L:(s + 1) * L], negs[s * L * n_neg:(s + 1) * L * n_neg],
                            alphas[s:s + 1], OConfig(**cfg))
    with fw.Trainer(fw.TrainConfig(deterministic=0, hot_rows=0, **cfg, **kn), text8.counts) as t:
        t.set_model(gi0, go0)
        for s in range(n):
            o = offsets[s:s + 2] - offsets[s]
            t.train_sentences(o, ids[s * L:(s + 1) * L], negs[s * L * n_neg:(s + 1) * L * n_neg], alphas[s:s + 1],
                              serial=False)
        gi, go = t.get_model()
    ei = np.linalg.norm((gi - ri).astype(np.float64)) / np.linalg.norm((ri - gi0).astype(np.float64))
    eo = np.linalg.norm((go - ro).astype(np.float64)) / np.linalg.norm((ro - go0).astype(np.float64))
    print(f"{mode} d={dim} {name}: relative update error input {ei:.2e} output {eo:.2e} (bound {bound:.0e})")
    assert ei <= bound and eo <= bound
