"""One traced e2e epoch (FW2V_TRACE timeline) on the text8 shape."""
import os, sys
os.environ["FW2V_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07743_b200 as fw
c = fw.synth_zipf(**fw.TEXT8_SHAPE)
cfg = fw.TrainConfig(dim=128, epochs=1, workers=int(os.environ.get("CHUNKS", "64")), streams=16, deterministic=0, reuse_mode="window_snapshot", sampler="alias")
with fw.Trainer(cfg, c.counts) as t:
    for _ in range(3):
        rep = t.train_corpus(c)
        print(f"e2e {rep.words_trained / rep.wall_seconds / 1e6:.1f} Mw/s  wall {rep.wall_seconds*1e3:.2f} ms", flush=True)
