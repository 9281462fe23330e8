"""Experiment: Zipf vs uniform corpus/negatives through K1s (hot-row contention test)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07743_b200 as fw
for name, s, power, sub in [("zipf", 1.0, 0.75, 1e-4), ("zipf-nosub", 1.0, 0.75, 0.0), ("uniform-neg", 1.0, 0.0, 1e-4), ("uniform", 0.0, 0.0, 1e-4)]:
    c = fw.synth_zipf(types=71291, tokens=16718845, s=s)
    cfg = fw.TrainConfig(dim=128, epochs=1, workers=16, batch_sentences=10000, deterministic=0, reuse_mode="window_snapshot", table_power=power, subsample=sub)
    with fw.Trainer(cfg, c.counts) as t:
        plan = t.plan_epoch(c, 0)
        secs = [plan.run()[0] for _ in range(3)]
        print(f"{name}: words={plan.words} {plan.words/min(secs)/1e6:.1f} Mwords/s", flush=True)
        plan.close()
