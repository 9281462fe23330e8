"""One bench step (text8 shape, bench.py's default knobs) between
cuProfilerStart/Stop, for `ncu --profile-from-start off`: the launch list of
exactly the launches bench.py times (64 plan batches on 16 x 2 streams, alias
sampler, hot-row replicas).
usage: python tools/ncu_bench_step.py [window_snapshot|lifetime] [workload text8|1bw] [dim]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "window_snapshot"
workload = sys.argv[2] if len(sys.argv) > 2 else "text8"
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 128
shape = fw.TEXT8_SHAPE if workload == "text8" else fw.ONEBW_SHAPE
corpus = fw.synth_zipf(**shape)
cfg = fw.TrainConfig(dim=dim, window=5, negatives=5, epochs=2, workers=64, streams=16, batch_sentences=10000,
                     subsample=1e-4, seed=1, deterministic=0, reuse_mode=mode, sampler="alias", l1_refresh_log2=5,
                     hot_rows=64, hot_merge=0)
# (hot_merge=0: ncu serialises kernels, so the live merge block, which runs beside the
# training kernels, would spin alone until its time cap; the K1s launches are the same.)
cuda = C.CDLL("libcuda.so.1")
with fw.Trainer(cfg, corpus.counts) as t:
    plan = t.plan_epoch(corpus, 0)
    plan.run()  # warm-up (not profiled)
    cuda.cuProfilerStart()
    secs, ctr = plan.run()
    cuda.cuProfilerStop()
    print(f"words {plan.words} launches {plan.batches} seconds {secs:.6f}", flush=True)
    plan.close()
