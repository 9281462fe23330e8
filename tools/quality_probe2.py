"""Snapshot vs lifetime semantics: serial reference runs and B200 Hogwild on planted + text8-shaped corpora."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2312_07743_b200 as fw
from oracle.oracle import Oracle, TrainConfig as RConfig
from test_quality import planted_corpus, CFG, _eval
from helpers import sgns_loss
ref = Oracle("ref")
counts, offsets, ids, wt = planted_corpus()
for mode in ["lifetime", "window_snapshot"]:
    rin, rout, rep = ref.train(counts, offsets, ids, RConfig(workers=1, reuse_mode=mode, **CFG))
    print(f"planted ref serial {mode}: {_eval(rin, rout, offsets, ids, counts, wt)}", flush=True)
c = fw.synth_zipf(**fw.TEXT8_SHAPE).head(3000)
p = c.counts.astype(np.float64) ** 0.75
negs = np.random.default_rng(5).choice(len(c.counts), len(c.ids) * 5, p=p / p.sum()).astype(np.int32)
T8 = dict(dim=128, window=5, negatives=5, epochs=3, batch_sentences=1000, subsample=1e-4, seed=1)
def ev(i, o): return sgns_loss(i, o, c.offsets, c.ids, negs, wf=3, n_neg=5, max_pairs=200_000)
for mode, w in [("lifetime", 16), ("window_snapshot", 16)]:
    t = time.time(); rin, rout, rep = ref.train(c.counts, c.offsets, c.ids, RConfig(workers=w, reuse_mode=mode, **T8))
    print(f"t8 ref {mode} w{w}: loss {ev(rin, rout):.4f} ({time.time()-t:.1f}s)", flush=True)
for mode in ["lifetime", "window_snapshot"]:
    for l1 in [0, 5]:
        with fw.Trainer(fw.TrainConfig(workers=16, deterministic=0, reuse_mode=mode, l1_refresh_log2=l1, **T8), c.counts) as t:
            t.train_corpus(c); gi, go = t.get_model()
        print(f"t8 ours {mode} l1={l1}: loss {ev(gi, go):.4f}", flush=True)
