"""Experiment: K1s memory-path flags on the text8-shaped Zipf corpus."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07743_b200 as fw
c = fw.synth_zipf(**fw.TEXT8_SHAPE)
for flags in [int(x, 0) for x in sys.argv[1].split(",")]:
    os.environ["FW2V_K1_FLAGS"] = str(flags)
    cfg = fw.TrainConfig(dim=128, epochs=1, workers=16, batch_sentences=10000, deterministic=0, reuse_mode="window_snapshot")
    with fw.Trainer(cfg, c.counts) as t:
        plan = t.plan_epoch(c, 0)
        secs = [plan.run()[0] for _ in range(3)]
        print(f"flags={flags:#x}: {plan.words/min(secs)/1e6:.1f} Mwords/s", flush=True)
        plan.close()
