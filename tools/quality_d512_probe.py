import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2312_07743_b200 as fw
from test_quality import planted_corpus, _eval, CFG
from oracle.oracle import Oracle, TrainConfig as RConfig
counts, offsets, ids, wt = planted_corpus()
ref = Oracle("ref")
rin, rout, _ = ref.train(counts, offsets, ids, RConfig(workers=os.cpu_count() or 4, dim=512, **CFG))
print("ref", _eval(rin, rout, offsets, ids, counts, wt), flush=True)
for mode in ("window_snapshot", "lifetime"):
    for lanes in (0, 32):
        for extra in ({}, {"hot_rows": 0}, {"max_inflight": 512}):
            cfg = fw.TrainConfig(workers=16, deterministic=0, reuse_mode=mode, dim=512, k1_lanes=lanes, **extra, **CFG)
            with fw.Trainer(cfg, counts) as t:
                t.train_corpus(fw.Corpus(counts, offsets, ids))
                gin, gout = t.get_model()
            print(mode, "lanes", lanes, extra, _eval(gin, gout, offsets, ids, counts, wt), flush=True)
