"""Shared fixtures: small corpora in the shapes the reference tests use
(test_trainer.cpp:86-121) and a numpy SGNS loss evaluator."""
from __future__ import annotations

import numpy as np


def random_corpus(n_sentences, max_len, types, seed, min_len=1):
    """Random ids with duplicates and collisions (test_trainer.cpp:108-121 shape).
    Counts are strictly decreasing in id so any vocabulary builder keeps id order."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(min_len, max_len + 1, n_sentences)
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    ids = rng.integers(0, types, int(offsets[-1])).astype(np.int32)
    counts = (100 + types - np.arange(types)).astype(np.uint64)
    return counts, offsets, ids


def distinct_corpus(n_sentences, sentence_len, seed):
    """Pairwise-distinct tokens per sentence (test_trainer.cpp:86-106 shape)."""
    rng = np.random.default_rng(seed)
    types = sentence_len * 4
    ids = np.concatenate([rng.permutation(types)[:sentence_len] for _ in range(n_sentences)]).astype(np.int32)
    offsets = (np.arange(n_sentences + 1) * sentence_len).astype(np.uint64)
    counts = (100 + types - np.arange(types)).astype(np.uint64)
    return counts, offsets, ids


def fixed_negatives(n_words, n_neg, vocab, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, vocab, n_words * n_neg).astype(np.int32)


def sgns_loss(inp, out, offsets, ids, negs, wf, n_neg, max_pairs=200_000, seed=0, split=None):
    """Mean SGNS objective over (context, target, negatives) triples of a fixed
    sample (SURVEY.md §7 hard part 7): -log s(c.t) - sum_n log s(-c.n), with c
    from the input matrix and t, n from the output matrix."""
    rng = np.random.default_rng(seed)
    n_sent = len(offsets) - 1
    trip_c, trip_t, trip_n = [], [], []
    while len(trip_c) < max_pairs:
        s = int(rng.integers(0, n_sent))
        b, e = int(offsets[s]), int(offsets[s + 1])
        L = e - b
        if L < 2:
            continue
        i = int(rng.integers(0, L))
        lo, hi = max(0, i - wf), min(L - 1, i + wf)
        j = int(rng.integers(lo, hi + 1))
        if j == i:
            continue
        trip_c.append(ids[b + j])
        trip_t.append(ids[b + i])
        trip_n.append(negs[(b + i) * n_neg:(b + i + 1) * n_neg])
    c = inp[np.array(trip_c)].astype(np.float64)
    t = out[np.array(trip_t)].astype(np.float64)
    n = out[np.array(trip_n)].astype(np.float64)
    ls = lambda x: -np.logaddexp(0.0, -x)  # noqa: E731  log sigmoid
    pos = ls(np.einsum("ij,ij->i", c, t))
    neg = ls(-np.einsum("ij,ikj->ik", c, n)).sum(axis=1)
    per = -(pos + neg)
    if split is not None:
        # (loss over triples whose target id < split, loss over the rest)
        hot = np.array(trip_t) < split
        return float(per[hot].mean()), float(per[~hot].mean())
    return float(per.mean())
