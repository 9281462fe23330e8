"""Scratch throughput probe: device-resident text8-shaped epoch through K1 shapes."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2312_07743_b200 as fw

t0 = time.time()
c = fw.synth_zipf(**fw.TEXT8_SHAPE)
print(f"corpus {time.time()-t0:.2f}s sentences={c.n_sentences} tokens={len(c.ids)}", flush=True)
dims = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["128"])]
for dim in dims:
    for lanes in ([0, 16] if dim == 128 else [0]):
        for S, mode in [(1000, "lifetime"), (1000, "window_snapshot"), (10000, "window_snapshot")]:
            cfg = fw.TrainConfig(dim=dim, epochs=1, workers=16, batch_sentences=S, deterministic=0, k1_lanes=lanes, reuse_mode=mode)
            with fw.Trainer(cfg, c.counts) as t:
                t0 = time.time()
                plan = t.plan_epoch(c, 0)
                tp = time.time() - t0
                secs = []
                for r in range(4):
                    s, ctr = plan.run()
                    secs.append(s)
                best = min(secs[1:])
                print(f"{mode} dim={dim} lanes={lanes or 'auto'} S={S} words={plan.words} plan={tp:.2f}s "
                      f"runs={[round(x*1e3,2) for x in secs]} ms -> {plan.words/best/1e6:.1f} Mwords/s "
                      f"({plan.words*(8*dim*7+24)/best/1e9:.0f} GB/s algorithmic)", flush=True)
                plan.close()
    # e2e through the host pipeline
    cfg = fw.TrainConfig(dim=dim, epochs=1, workers=16, batch_sentences=1000, deterministic=0, reuse_mode="window_snapshot")
    with fw.Trainer(cfg, c.counts) as t:
        rep = t.train_corpus(c)
        print(f"e2e dim={dim}: {rep.words_trained/rep.wall_seconds/1e6:.1f} Mwords/s wall={rep.wall_seconds:.3f}s "
              f"batching={rep.batching_words_per_sec/1e6:.1f} Mw/s/thread", flush=True)
