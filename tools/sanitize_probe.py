"""Small runs of every kernel family for compute-sanitizer (tests/test_sanitizers.py):
K2 (serial exact, all reuse modes), K1s in both update orders with the bench's
knobs and with the exact knobs, multi-chunk (N=15) and d=512 two-warp shapes,
the hot-row replica sync, init_model and the replica merge kernels.
usage: compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402


def corpus(n, max_len, types, seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, max_len + 1, n)
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    ids = rng.integers(0, types, int(offsets[-1])).astype(np.int32)
    counts = (100 + types - np.arange(types)).astype(np.uint64)
    return fw.Corpus(counts, offsets, ids)


def main():
    c = corpus(24, 40, 60, 1)
    runs = []
    for mode in ("lifetime", "window", "none", "window_snapshot"):
        runs.append(dict(dim=32, workers=1, reuse_mode=mode))  # K2
    for mode in ("lifetime", "window_snapshot"):
        for dim, neg, window in ((128, 5, 5), (300, 5, 5), (512, 5, 5), (128, 15, 5), (64, 5, 9)):
            runs.append(dict(dim=dim, negatives=neg, window=window, workers=4, deterministic=0, reuse_mode=mode,
                             sampler="alias", hot_rows=8))  # bench knobs
            runs.append(dict(dim=dim, negatives=neg, window=window, workers=4, deterministic=0, reuse_mode=mode,
                             fast_sigmoid=False, l1_refresh_log2=0, delta_writeback=0, hot_rows=0))  # exact knobs
    for kw in runs:
        kw.setdefault("negatives", 5)
        kw.setdefault("window", 5)
        cfg = fw.TrainConfig(epochs=1, batch_sentences=7, table_size=10007, subsample=1e-2, seed=3, **kw)
        with fw.Trainer(cfg, c.counts) as t:
            t.train_corpus(c)
            gi, go = t.get_model()
        assert np.isfinite(gi).all() and np.isfinite(go).all(), kw
    # replica merge kernels (peer path: two replicas on one device)
    cfg = fw.TrainConfig(dim=32, epochs=1, workers=4, deterministic=0, batch_sentences=7, table_size=10007)
    ts = [fw.Trainer(cfg, c.counts) for _ in range(2)]
    fw.train_corpus_multi(ts, c, average_words=100)
    fw.average(ts)
    for t in ts:
        t.close()
    print(f"sanitize probe ok: {len(runs)} training runs + replica merge")


if __name__ == "__main__":
    main()
