"""SURVEY §8(d) sweep on the 1bw shape: d x window x negatives (x S at d=128),
both reuse modes, device-resident epochs (fw2v_plan_epoch / plan.run), 1 B200.

Prints one line per config: Mwords/s (median of 2 timed epochs after 1 warm-up)
and the algorithmic HBM fraction B(d,N) x words/s / measured peak.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07743_b200 as fw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0

t0 = time.time()
corpus = fw.synth_zipf(**fw.ONEBW_SHAPE)
print(f"# 1bw-shaped corpus: {int(corpus.offsets[-1])} tokens, {len(corpus.counts)} types, "
      f"built in {time.time() - t0:.1f} s; HBM peak {peak} GB/s", flush=True)

avail_gb = 0.0
with open("/proc/meminfo") as f:
    for line in f:
        if line.startswith("MemAvailable:"):
            avail_gb = int(line.split()[1]) / 2**20
print(f"# host MemAvailable {avail_gb:.0f} GB", flush=True)

modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["window_snapshot", "lifetime"]
dims = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [64, 128, 256, 512]
grid = [(d, w, n, 10000) for d in dims for w in (2, 5, 8) for n in (5, 15)]
if 128 in dims:
    grid += [(128, 5, 5, 1000), (128, 5, 5, 50000)]
for mode in modes:
    for d, w, n, S in grid:
        if n == 15 and avail_gb < 120:  # the host-side plan of an N=15 epoch is ~34 GB
            print(f"{mode:15s} d={d:3d} W={w} N={n:2d} S={S:5d}  skipped: host memory", flush=True)
            continue
        cfg = fw.TrainConfig(dim=d, window=w, negatives=n, epochs=3, workers=64, streams=16, batch_sentences=S,
                             subsample=1e-4, seed=1, deterministic=0, reuse_mode=mode, sampler="alias")
        try:
            with fw.Trainer(cfg, corpus.counts) as t:
                plan = t.plan_epoch(corpus, 0)
                secs = []
                for k in range(3):
                    s, _ = plan.run()
                    if k:
                        secs.append(s)
                words = plan.words
                plan.close()
            rate = words / min(secs)
            bpw = 8 * d * (n + 2) + 4 * (n + 1)
            print(f"{mode:15s} d={d:3d} W={w} N={n:2d} S={S:5d}  {rate / 1e6:8.1f} Mw/s  "
                  f"frac {rate * bpw / 1e9 / peak:.3f}  ({words / 1e6:.0f} M words/epoch)", flush=True)
        except Exception as e:  # keep sweeping
            print(f"{mode:15s} d={d:3d} W={w} N={n:2d} S={S:5d}  failed: {e}", flush=True)
