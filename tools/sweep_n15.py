"""1bw shape, N=15 (and N=5 control) at d=64/128/256, both orders: device-resident epochs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07743_b200 as fw
corpus = fw.synth_zipf(**fw.ONEBW_SHAPE)
for mode in ("window_snapshot", "lifetime"):
    for d in (64, 128, 256):
        for w, n in ((2, 15), (5, 15), (8, 15), (5, 5)):
            cfg = fw.TrainConfig(dim=d, window=w, negatives=n, epochs=3, workers=64, streams=16, subsample=1e-4,
                                 deterministic=0, reuse_mode=mode, sampler="alias")
            with fw.Trainer(cfg, corpus.counts) as t:
                plan = t.plan_epoch(corpus, 0)
                secs = [plan.run()[0] for _ in range(3)][1:]
                words = plan.words
                plan.close()
            rate = words / min(secs)
            bpw = 8 * d * (n + 2) + 4 * (n + 1)
            print(f"{mode:15s} d={d:3d} W={w} N={n:2d}  {rate / 1e6:8.1f} Mw/s  frac {rate * bpw / 1e9 / 6550.1:.3f}", flush=True)
