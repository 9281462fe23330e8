"""Small driver for ncu captures: text8-shaped epoch plan, run twice.
usage: ncu_probe.py [mode] [batch_sentences] [dim] [workers]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07743_b200 as fw
mode = sys.argv[1] if len(sys.argv) > 1 else "window_snapshot"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 128
workers = int(sys.argv[4]) if len(sys.argv) > 4 else 16
c = fw.synth_zipf(**fw.TEXT8_SHAPE)
cfg = fw.TrainConfig(dim=dim, epochs=1, workers=workers, batch_sentences=S, deterministic=0, reuse_mode=mode)
with fw.Trainer(cfg, c.counts) as t:
    plan = t.plan_epoch(c, 0)
    for _ in range(2):
        s, _ = plan.run()
        print(f"{mode} {plan.words/s/1e6:.1f} Mwords/s", flush=True)
    plan.close()
