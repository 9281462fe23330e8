"""Per-epoch times of 20-epoch fw2v_train_corpus calls (reference-default shape:
workers = 0) with the live hot-row merge on / off (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402

corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
hm_list = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 0, 1]
for hm in hm_list:
    cfg = fw.TrainConfig(dim=128, window=5, negatives=5, epochs=20, workers=0, batch_sentences=10000, subsample=1e-4,
                         seed=1, reuse_mode="window_snapshot", sampler="alias", deterministic=0, hot_merge=hm)
    t0 = time.perf_counter()
    with fw.Trainer(cfg, corpus.counts) as t:
        t1 = time.perf_counter()
        rep = t.train_corpus(corpus)
        t2 = time.perf_counter()
    t3 = time.perf_counter()
    eps = sorted(e["seconds"] * 1e3 for e in rep.epochs)
    print(f"hot_merge={hm}: create {1e3 * (t1 - t0):.0f} ms train {1e3 * (t2 - t1):.0f} ms close {1e3 * (t3 - t2):.0f} ms; "
          f"epoch ms min {eps[0]:.2f} med {eps[len(eps) // 2]:.2f} max {eps[-1]:.2f}", flush=True)
