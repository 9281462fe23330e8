"""Loss / recall@10 of reference (various workers) vs B200 trainers on the planted corpus."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2312_07743_b200 as fw
from oracle.oracle import Oracle, TrainConfig as RConfig
from test_quality import planted_corpus, CFG, _eval
counts, offsets, ids, wt = planted_corpus()
ref = Oracle("ref")
for w in [1, 16]:
    t = time.time(); rin, rout, rep = ref.train(counts, offsets, ids, RConfig(workers=w, **CFG))
    print(f"ref workers={w}: loss/recall {_eval(rin, rout, offsets, ids, counts, wt)} words={rep.words_trained} ({time.time()-t:.1f}s)", flush=True)
for mode, det, l1, streams in [("lifetime", 1, 0, 1), ("lifetime", 0, 0, 16), ("window_snapshot", 0, 0, 16), ("window_snapshot", 0, 5, 16)]:
    cfg = fw.TrainConfig(workers=streams, deterministic=det, reuse_mode=mode, l1_refresh_log2=l1, **CFG)
    with fw.Trainer(cfg, counts) as t:
        rep = t.train_corpus(fw.Corpus(counts, offsets, ids)); gin, gout = t.get_model()
    print(f"ours {mode} det={det} l1={l1} streams={streams}: {_eval(gin, gout, offsets, ids, counts, wt)}", flush=True)
