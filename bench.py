#!/usr/bin/env python
"""FULL-W2V B200 benchmark: trained words/s at d=128 w=5 neg=5 (BASELINE.json).

Workload (config.workload): the text8-shaped synthetic Zipf corpus of
BASELINE.md §2 (71,291 ranks, 16,718,845 tokens, 1000-token sentences,
subsample 1e-4, window 5 -> W_f 3, 5 negatives, d 128, S 10,000 sentences per
producer batch, 16 producer streams), trained with the FULL-W2V
independent-negatives window kernel K1s (reference ReuseMode::window_snapshot,
trainer.cpp:158-205) under Hogwild.

One step = one epoch over the corpus. `value` is device-resident: the epoch's
batches (ids, negatives, alpha) are assembled once into HBM by the host batcher
(fw2v_plan_epoch) and each step launches only the training kernels, timed with
CUDA events on the launching streams. `e2e` is the same metric through the
reference-facing C-ABI (fw2v_train_corpus): per step the host batching threads
subsample, draw negatives, fill pinned buffers, copy H2D and launch; the D2H is
the per-stream counter read-back. Inputs per step (238 MB id+negative stream)
exceed the 126 MB L2, so no flush is needed between steps; the 73 MB model is
L2-resident by design, which is the point of the kernel.

Multi-GPU (torchrun, one process per GPU): weak scaling, each rank trains a
text8-shaped shard with its own RNG streams and the replicas are averaged
after every step with an NCCL all-reduce (ncclAvg) over the model tensors;
timing is the max over ranks.

--impl reference times the reference CPU trainer (ringvec::train compiled from
/root/reference by oracle/Makefile into oracle/_ref) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trained words/sec at d=128 w=5 neg=5 (1/2/4/8 B200) + % HBM roofline"
UNIT = "words/s"


def algorithmic_bytes_per_word(d, n):
    """Lifetime-mode model traffic per trained word (traffic.cpp:35-42):
    (N+1) sample reads + writes and 1 context read + write of 4d bytes, plus ids/negatives."""
    return 8 * d * (n + 2) + 4 * (n + 1)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sms, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sms.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sms:
            return None
        sms.sort()
        return {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_

        n_dev = torch.cuda.device_count()
        if n_dev >= world:
            torch.cuda.set_device(local)
            dist_.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # Functional check of the multi-rank path on a box with fewer GPUs than
            # ranks (ranks share devices, gloo all-reduce): numbers are not a measurement.
            local = local % max(n_dev, 1)
            torch.cuda.set_device(local)
            dist_.init_process_group("gloo")
            print(f"[bench] {world} ranks on {n_dev} GPU(s): gloo, functional check only", file=sys.stderr)
        dist = dist_
    return world, rank, local, dist


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, world, rank):
    """Reference CPU trainer (oracle/_ref, compiled from /root/reference) on host cores."""
    if rank != 0:
        return
    import numpy as np

    import paper_2312_07743_b200 as fw
    from oracle.oracle import Oracle, TrainConfig as RConfig

    ref = Oracle("ref")
    shape = fw.TEXT8_SHAPE if args.workload == "text8" else fw.ONEBW_SHAPE
    corpus = fw.synth_zipf(**shape)
    sample = corpus.head(args.ref_sentences)
    cores = cpu_cores()
    cfg = RConfig(dim=args.dim, window=args.window, negatives=args.negatives, epochs=1, workers=cores,
                  batch_sentences=args.batch_sentences, subsample=1e-4, seed=1)
    rates = []
    for step in range(args.warmup + args.steps):
        _, _, rep = ref.train(sample.counts, sample.offsets, sample.ids, cfg)
        if step >= args.warmup:
            rates.append(rep.epoch_words_per_sec[0])
    value = float(np.median(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"{args.workload}-shaped Zipf corpus, bounded sample of {args.ref_sentences} sentences",
                   "dim": args.dim, "window": args.window, "negatives": args.negatives, "subsample": 1e-4,
                   "reuse_mode": "lifetime (reference default)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"first {args.ref_sentences} sentences ({int(sample.offsets[-1])} tokens) of the "
                                   f"{args.workload}-shaped corpus, 1 epoch per step, workers={cores}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local, dist):
    import numpy as np
    import torch

    import paper_2312_07743_b200 as fw

    shape = fw.TEXT8_SHAPE if args.workload == "text8" else fw.ONEBW_SHAPE
    corpus = fw.synth_zipf(**shape)
    cfg = fw.TrainConfig(dim=args.dim, window=args.window, negatives=args.negatives, epochs=max(1, args.steps),
                         workers=args.chunks, streams=args.streams, batch_sentences=args.batch_sentences,
                         subsample=1e-4,
                         seed=1 + rank, deterministic=0, reuse_mode=args.reuse_mode, device=local,
                         sampler=args.sampler, l1_refresh_log2=args.l1_refresh_log2, k1_lanes=args.k1_lanes)
    trainer = fw.Trainer(cfg, corpus.counts)
    model = None
    if dist is not None:
        # Replicas live in torch tensors so NCCL can average them in place.
        v, stride = trainer.vocab, trainer.stride
        model = torch.zeros((2, v, stride), dtype=torch.float32, device=f"cuda:{local}")
        torch.cuda.synchronize()
        trainer.attach_model(model[0].data_ptr(), model[1].data_ptr())
        trainer.init_model(1)  # identical initial replicas on every rank

    plan = trainer.plan_epoch(corpus, 0)
    words_per_step = plan.words
    n_launches = plan.batches

    averager = None
    if dist is not None:
        from paper_2312_07743_b200.dist import ReplicaAverager

        averager = ReplicaAverager(model)

    def average():
        if averager is not None:
            torch.cuda.synchronize()
            averager.average()  # one in-place NCCL all-reduce (AVG) over syn0 + syn1
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        plan.run()
        average()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    step_secs = []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s, ctr = plan.run()
            step_secs.append(s)
            average()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if dist is not None:
        dist.barrier()
    dev_time = float(sum(step_secs))
    t_max = dev_time
    if dist is not None:
        t = torch.tensor([dev_time], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    total_words = words_per_step * args.steps * world
    value = total_words / t_max
    ms_per_step = 1e3 * t_max / args.steps
    plan.close()

    # e2e: the same metric through fw2v_train_corpus (host batching + pinned H2D).
    e2e = None
    if not args.no_e2e:
        ecfg = fw.TrainConfig(**{**cfg.__dict__, "epochs": 1})
        with fw.Trainer(ecfg, corpus.counts) as et:
            et.train_corpus(corpus)  # warm-up epoch (allocates pinned buffers)
            e_words, e_secs, h2d, bwps = 0, 0.0, 0, 0.0
            for _ in range(max(1, min(args.steps, 3))):
                if dist is not None:
                    dist.barrier()
                rep = et.train_corpus(corpus)
                e_words += rep.words_trained
                e_secs += rep.wall_seconds
                h2d = rep.h2d_bytes
                bwps = rep.batching_words_per_sec
            e_rate = e_words / e_secs
            if dist is not None:
                t = torch.tensor([e_secs], device=f"cuda:{local}", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                e_rate = e_words * world / float(t.item())
            e2e = {"value": e_rate, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": 64 * args.streams,
                   "path": "fw2v_train_corpus (C-ABI): host batching threads -> pinned -> H2D -> K1s",
                   "host_batching_words_per_sec_per_thread": bwps, "batching_threads": args.streams}

    peak, peak_src = load_peaks()
    bpw = algorithmic_bytes_per_word(args.dim, args.negatives)
    achieved = words_per_step * bpw / (t_max / args.steps) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_k1s_summary.json")
    if os.path.exists(prof):
        with open(prof) as f:
            j = json.load(f)
        traffic = j.get("dram_bytes_per_launch")
    clocks = clk.summary()
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_baseline = cpu_baseline_leg(args, corpus)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": f"{args.workload}-shaped Zipf corpus ({shape['types']} ranks, "
                                   f"{shape['tokens']} tokens, 1000-token sentences), 1 epoch per step",
                       "dim": args.dim, "window": args.window, "negatives": args.negatives, "subsample": 1e-4,
                       "words_per_step_per_gpu": words_per_step, "batch_sentences": args.batch_sentences,
                       "streams": args.streams, "chunks": args.chunks, "reuse_mode": args.reuse_mode,
                       "kernel": "K1s (FULL-W2V independent negatives, Hogwild)", "sampler": args.sampler,
                       "l1_refresh_log2": args.l1_refresh_log2,
                       "parallelism": f"dp{world} replicas + NCCL avg per step" if world > 1 else "single GPU",
                       "l2_policy": "inputs (238 MB id/negative stream per step) > 126 MB L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_word": bpw,
                         "note": "algorithmic lifetime-mode bytes/word x words/s; the model is L2-resident "
                                 "so frac can exceed 1 (ncu: ~124 B of DRAM traffic per word). The kernel is "
                                 "issue/L1-bound: 492 warp-instructions per word against an FFMA2 floor of 216, "
                                 "issue 53%, FMA pipe 53%, L1 wavefronts 73% (profiles/r01l_k1s_snapshot_quick.txt)"},
            "e2e": e2e, "gpu_launches": (n_launches + (2 if cfg.hot_rows > 0 else 0)) * args.steps, "clocks": clocks,
            "wall_s_timed": wall,
        }
        if cpu_baseline is not None:
            line["cpu_baseline"] = cpu_baseline
        print(json.dumps(line), flush=True)
    trainer.close()
    if dist is not None:
        dist.destroy_process_group()


def cpu_baseline_leg(args, corpus):
    from oracle.oracle import Oracle, available, TrainConfig as RConfig

    kind = "reference" if available("ref") else "port"
    o = Oracle("ref" if kind == "reference" else "oracle")
    sample = corpus.head(args.ref_sentences)
    cores = cpu_cores() if kind == "reference" else 1
    cfg = RConfig(dim=args.dim, window=args.window, negatives=args.negatives, epochs=1, workers=cores,
                  batch_sentences=args.batch_sentences, subsample=1e-4, seed=1)
    _, _, rep = o.train(sample.counts, sample.offsets, sample.ids, cfg)
    return {"value": rep.epoch_words_per_sec[0], "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"first {args.ref_sentences} sentences ({int(sample.offsets[-1])} tokens) of the corpus, "
                      f"1 epoch, reference lifetime mode, workers={cores}"}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["text8", "1bw"], default="text8")
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--window", type=int, default=5)
    ap.add_argument("--negatives", type=int, default=5)
    ap.add_argument("--batch-sentences", type=int, default=10000)
    ap.add_argument("--streams", type=int, default=16, help="batching threads = CUDA streams")
    ap.add_argument("--chunks", type=int, default=64,
                    help="corpus chunks (TrainConfig.workers: the reference's producer partition and RNG streams)")
    ap.add_argument("--reuse-mode", default="window_snapshot")
    ap.add_argument("--sampler", default="alias", choices=["reference", "alias"])
    ap.add_argument("--l1-refresh-log2", type=int, default=5)
    ap.add_argument("--k1-lanes", type=int, default=0, help="lanes per sentence (0 = auto)")
    ap.add_argument("--ref-sentences", type=int, default=4000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        if dist is not None:
            dist.destroy_process_group()
        return
    run_ours(args, world, rank, local, dist)


if __name__ == "__main__":
    main()
