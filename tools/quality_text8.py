"""Quality probe on the text8-shaped (or, with FW2V_SHAPE=1bw, the 1bw-shaped) Zipf
corpus: SGNS loss of the reference CPU trainer vs the B200 trainer under several
Hogwild settings.
usage: python tools/quality_text8.py [dim] [epochs] [config ...]   config = key=value,key=value"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2312_07743_b200 as fw  # noqa: E402
from helpers import sgns_loss  # noqa: E402
from oracle.oracle import Oracle, TrainConfig as RConfig  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 128
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
configs = sys.argv[3:] or ["reuse_mode=window_snapshot"]
c = fw.synth_zipf(**(fw.ONEBW_SHAPE if os.environ.get("FW2V_SHAPE") == "1bw" else fw.TEXT8_SHAPE))
counts, offsets, ids = c.counts, c.offsets, c.ids
p = counts.astype(np.float64) ** 0.75
negs = np.random.default_rng(5).choice(len(counts), 400_000 * 5, p=p / p.sum()).astype(np.int32)
sub_off = offsets[: 401].copy()  # held-out sample: first 400 sentences' positions
base = dict(dim=dim, window=5, negatives=5, epochs=epochs, batch_sentences=10000, subsample=1e-4, seed=1)


def loss(inp, out):
    return sgns_loss(inp, out, sub_off, ids[: int(sub_off[-1])], negs, wf=3, n_neg=5, max_pairs=100_000)


t = time.time()
rin, rout, rrep = Oracle("ref").train(counts, offsets, ids, RConfig(workers=os.cpu_count() or 8, **base))
print(f"reference lifetime workers={os.cpu_count()}: loss {loss(rin, rout):.4f}  ({time.time() - t:.1f}s)", flush=True)
for spec in configs:
    kw = dict(base, workers=16, deterministic=0)
    for item in spec.split(","):
        k, v = item.split("=")
        kw[k] = type(getattr(fw.TrainConfig(), k))(v) if not isinstance(getattr(fw.TrainConfig(), k), bool) else v not in ("0", "false", "False")
    with fw.Trainer(fw.TrainConfig(**kw), counts) as tr:
        rep = tr.train_corpus(c)
        gin, gout = tr.get_model()
    bad = int((~np.isfinite(gin)).sum() + (~np.isfinite(gout)).sum())
    print(f"{spec}: loss {loss(gin, gout):.4f}  max|out| {np.abs(gout).max():.3g}  nonfinite {bad}  "
          f"{rep.words_trained / rep.wall_seconds / 1e6:.0f} Mw/s e2e", flush=True)
