"""W=5, N=11/15 throughput on the 1bw shape (used to choose 8- vs 6-sample chunks; the FW2V_K1S_NC8 switch it compared is gone: 8-sample chunks are now picked automatically)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07743_b200 as fw
corpus = fw.synth_zipf(**fw.ONEBW_SHAPE)
tag = "nc8" if os.environ.get("FW2V_K1S_NC8") else "nc6"
for mode in ("window_snapshot", "lifetime"):
    for d in (64, 128, 256, 512):
        for n in (15, 11):
            cfg = fw.TrainConfig(dim=d, window=5, negatives=n, epochs=3, workers=64, streams=16, subsample=1e-4,
                                 deterministic=0, reuse_mode=mode, sampler="alias")
            with fw.Trainer(cfg, corpus.counts) as t:
                plan = t.plan_epoch(corpus, 0)
                secs = [plan.run()[0] for _ in range(3)][1:]
                words = plan.words
                plan.close()
            print(f"{tag} {mode:15s} d={d:3d} W=5 N={n:2d}  {words / min(secs) / 1e6:8.1f} Mw/s", flush=True)
