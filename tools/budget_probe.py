"""Hogwild in-flight budget on the text8 shape without hot-row replicas: SGNS loss
after 5 epochs vs the reference train() (oracle/_ref, all host cores), at the
automatic budget, fixed caps and unlimited, both update orders; plus e2e rate."""
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2312_07743_b200 as fw  # noqa: E402
from helpers import sgns_loss  # noqa: E402
from oracle.oracle import Oracle, TrainConfig as RConfig  # noqa: E402

c = fw.synth_zipf(**fw.TEXT8_SHAPE)
cfg = dict(dim=128, window=5, negatives=5, epochs=5, batch_sentences=10000, subsample=1e-4, seed=1)
p = c.counts.astype(np.float64) ** 0.75
negs = np.random.default_rng(5).choice(len(c.counts), 400_000 * 5, p=p / p.sum()).astype(np.int32)
off = c.offsets[:401].copy()


def loss(i, o):
    return sgns_loss(i, o, off, c.ids[: int(off[-1])], negs, wf=3, n_neg=5, max_pairs=100_000)


t0 = time.time()
rin, rout, _ = Oracle("ref").train(c.counts, c.offsets, c.ids, RConfig(workers=os.cpu_count() or 8, **cfg))
ref = loss(rin, rout)
print(f"reference loss {ref:.4f} ({time.time() - t0:.0f} s)", flush=True)
for mode in ("window_snapshot", "lifetime"):
    for mi in (0, 2960, 4000, -1):
        k = dict(workers=64, streams=16, sampler="alias", hot_rows=0, deterministic=0, max_inflight=mi,
                 divergence_guard=0)
        with fw.Trainer(fw.TrainConfig(reuse_mode=mode, **cfg, **k), c.counts) as t:
            t0 = time.perf_counter()
            rep = t.train_corpus(c)
            dt = time.perf_counter() - t0
            gi, go = t.get_model()
        g = loss(gi, go)
        print(f"{mode:16s} max_inflight {mi:5d}: loss {g:.4f} ({100 * (g / ref - 1):+.2f}%) "
              f"{rep.words_trained / dt / 1e6:.0f} Mw/s max|x| {max(np.abs(gi).max(), np.abs(go).max()):.3g}",
              flush=True)
