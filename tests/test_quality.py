"""Tier-2 parity (north_star): Hogwild runs on the B200 must match the reference
CPU trainer's final SGNS loss within 2% and recover its planted-neighbour
structure at equal recall@10.

Planted corpus (the shape of test_trainer.cpp:561-632, scaled up): T topics of
exclusive words plus a shared pool; each sentence draws 70% of its tokens
from one topic. Both trainers see the same corpus and config; the reference
runs lifetime mode with all host cores (oracle/_ref), ours runs the Hogwild
K1 (lifetime) and K1s (FULL-W2V independent negatives) kernels.
"""
import numpy as np
import pytest

from helpers import sgns_loss

pytestmark = pytest.mark.gpu
fw = pytest.importorskip("paper_2312_07743_b200")
from oracle.oracle import TrainConfig as RConfig  # noqa: E402

TOPICS, PER_TOPIC, SHARED = 100, 20, 100


def planted_corpus(n_sentences=12000, length=30, seed=20240811):
    rng = np.random.default_rng(seed)
    types = TOPICS * PER_TOPIC + SHARED
    topic = rng.integers(0, TOPICS, n_sentences)
    pick_topic = rng.random((n_sentences, length)) < 0.7
    tw = topic[:, None] * PER_TOPIC + rng.integers(0, PER_TOPIC, (n_sentences, length))
    sw = TOPICS * PER_TOPIC + rng.integers(0, SHARED, (n_sentences, length))
    ids = np.where(pick_topic, tw, sw).astype(np.int32).ravel()
    offsets = (np.arange(n_sentences + 1) * length).astype(np.uint64)
    # strictly decreasing counts keep vocabulary ids equal to generated ids
    counts = (10_000_000 - np.arange(types)).astype(np.uint64)
    return counts, offsets, ids


def recall_at_10(inp):
    words = TOPICS * PER_TOPIC
    v = inp[:words].astype(np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True) + 1e-12
    sim = v @ v.T
    np.fill_diagonal(sim, -np.inf)
    top = np.argpartition(-sim, 10, axis=1)[:, :10]
    same = (top // PER_TOPIC) == (np.arange(words)[:, None] // PER_TOPIC)
    return float(same.mean())


CFG = dict(dim=32, window=5, negatives=5, epochs=4, batch_sentences=500, subsample=0.0, table_size=1_000_003,
           alpha0=0.05, seed=3)


@pytest.fixture(scope="module")
def reference_run(ref):
    import os

    counts, offsets, ids = planted_corpus()
    inp, out, rep = ref.train(counts, offsets, ids, RConfig(workers=os.cpu_count() or 4, **CFG))
    return counts, offsets, ids, inp, out


def _eval(inp, out, offsets, ids, vocab):
    negs = np.random.default_rng(5).integers(0, vocab, len(ids) * 5).astype(np.int32)
    return sgns_loss(inp, out, offsets, ids, negs, wf=3, n_neg=5, max_pairs=100_000), recall_at_10(inp)


@pytest.mark.parametrize("mode", ["lifetime", "window_snapshot"])
@pytest.mark.parametrize("l1_refresh_log2", [0, 5])
def test_hogwild_quality_matches_reference(reference_run, mode, l1_refresh_log2):
    counts, offsets, ids, rin, rout = reference_run
    ref_loss, ref_recall = _eval(rin, rout, offsets, ids, len(counts))
    cfg = fw.TrainConfig(workers=16, deterministic=0, reuse_mode=mode, l1_refresh_log2=l1_refresh_log2, **CFG)
    with fw.Trainer(cfg, counts) as t:
        t.train_corpus(fw.Corpus(counts, offsets, ids))
        gin, gout = t.get_model()
    loss, recall = _eval(gin, gout, offsets, ids, len(counts))
    print(f"{mode} l1={l1_refresh_log2}: loss {loss:.4f} vs ref {ref_loss:.4f}; recall@10 {recall:.4f} vs {ref_recall:.4f}")
    assert abs(loss - ref_loss) / ref_loss <= 0.02
    assert recall >= ref_recall - 0.01
