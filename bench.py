#!/usr/bin/env python
"""FULL-W2V B200 benchmark: trained words/s at d=128 w=5 neg=5 (BASELINE.json).

Workload (config.workload): the text8-shaped synthetic Zipf corpus of
BASELINE.md §2 (71,291 ranks, 16,718,845 tokens, 1000-token sentences,
subsample 1e-4, window 5 -> W_f 3, 5 negatives, d 128, S 10,000 sentences per
producer batch) trained under Hogwild with the FULL-W2V independent-negatives
window kernel K1s (reference ReuseMode::window_snapshot, trainer.cpp:158-205).
One step = one epoch over the corpus.

* `value`: device-resident. The epoch's batches (ids, negatives, alpha) are
  assembled once into HBM (fw2v_plan_epoch); a step launches only the training
  kernels, timed with CUDA events on the launching streams.
* `e2e`: the same metric through the reference-facing C-ABI
  (fw2v_train_corpus): per step the host batching threads subsample, draw
  negatives, fill pinned buffers, copy H2D and launch; the D2H is the
  per-stream counter read-back.
* `lifetime`: the same two numbers in the reference's DEFAULT update order
  (ReuseMode::lifetime, config.hpp:25; sweep_samples trainer.cpp:133-154) —
  the like-for-like counterpart of the reference arm.
* `dropin_e2e`: whole `ringvec::train` calls through the C++ drop-in with the
  reference's default TrainConfig (workers = hardware threads) — context
  setup, batching, H2D, kernels, model readback — per update order.
Inputs per step (238 MB id+negative stream) exceed the 126 MB L2, so no flush
is needed between steps; the 73 MB model is L2-resident by design.

Multi-GPU (torchrun, one process per GPU): each rank holds a
replica and trains a contiguous shard of whole chunks (fw2v_plan_chunks /
fw2v_train_corpus_multi); the replicas are merged inside the timed region
every --average-words words per GPU and after every step with the library's
NCCL communicator (fw2v_comm_init_rank; ncclAllReduce over NVLink). text8:
weak scaling (world x text8 tokens, one text8-sized shard per GPU); 1bw: the
1bw-shaped corpus split across the ranks (strong scaling). Timing: max over
ranks.

--impl reference times the reference CPU trainer (ringvec::train compiled from
/root/reference by oracle/Makefile into oracle/_ref) on the host's hardware
threads over the same corpus, built by the reference itself
(Vocabulary::build, oracle/ref_capi.cpp ref_synth_corpus).
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
TEXT8 = dict(types=71_291, tokens=16_718_845)
ONEBW = dict(types=555_514, tokens=804_269_957)
PROFILE = os.path.join(ROOT, "profiles", "bench_roofline.json")


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


def load_profile():
    """ncu figures of the benched launches (tools/ncu_bench_step.py -> profiles/)."""
    if os.path.exists(PROFILE):
        with open(PROFILE) as f:
            return json.load(f)
    return {}


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
    dist, shared = None, False
    if world > 1:
        import torch
        import torch.distributed as dist_

        n_dev = torch.cuda.device_count()
        if n_dev >= world:
            torch.cuda.set_device(local)
            dist_.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # Functional check of the multi-rank path on a box with fewer GPUs than
            # ranks (ranks share devices, gloo exchange): numbers are not a measurement.
            local = local % max(n_dev, 1)
            torch.cuda.set_device(local)
            dist_.init_process_group("gloo")
            shared = True
            print(f"[bench] {world} ranks on {n_dev} GPU(s): gloo, functional check only", file=sys.stderr)
        dist = dist_
    return world, rank, local, dist, shared


def host_cores():
    """(physical cores, hardware threads) of this host (lscpu; affinity for threads)."""
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or 1
    phys = None
    try:
        out = subprocess.run(["lscpu", "-p=Core,Socket"], capture_output=True, text=True, timeout=10).stdout
        pairs = {ln for ln in out.splitlines() if ln and not ln.startswith("#")}
        phys = len(pairs) or None
    except (OSError, subprocess.SubprocessError):
        pass
    return phys or threads, threads


def shape_of(workload):
    return TEXT8 if workload == "text8" else ONEBW


def run_reference(args, world, rank):
    """The reference CPU trainer (oracle/_ref: ringvec::train compiled from
    /root/reference) on the host's hardware threads (TrainConfig.workers = 0,
    the reference default: hardware_concurrency), over the workload's corpus
    built by the reference itself; libfw2v is not loaded on this arm."""
    if rank != 0:
        return
    import numpy as np

    from oracle.oracle import Oracle, RefCorpus, TrainConfig as RConfig

    ref = Oracle("ref")
    shape = shape_of(args.workload)
    full = RefCorpus(ref, shape["types"], shape["tokens"])
    phys, threads = host_cores()
    cfg = RConfig(dim=args.dim, window=args.window, negatives=args.negatives, epochs=1, workers=0,
                  batch_sentences=args.batch_sentences, subsample=1e-4, seed=1)
    # Size the step: the full epoch if the whole run fits the budget, else the
    # first sentences that do (named in config.workload).
    corpus, sample = full, f"full {args.workload}-shaped epoch ({full.n_sentences} sentences)"
    probe = full.head(min(full.n_sentences, 2000))
    t0 = time.perf_counter()
    probe.train(cfg)
    per_sentence = (time.perf_counter() - t0) / probe.n_sentences
    budget = args.ref_budget_s / max(1, args.steps + args.warmup)
    if per_sentence * full.n_sentences > budget:
        n = max(200, int(budget / per_sentence))
        corpus = full.head(n)
        sample = f"first {n} of {full.n_sentences} sentences of the {args.workload}-shaped corpus"
    rates = []
    for step in range(args.warmup + args.steps):
        rep = corpus.train(cfg)
        if step >= args.warmup:
            rates.append(rep.epoch_words_per_sec[0])
    value = float(np.median(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"{args.workload}-shaped Zipf corpus, {sample}, 1 epoch per step",
                   "dim": args.dim, "window": args.window, "negatives": args.negatives, "subsample": 1e-4,
                   "reuse_mode": "lifetime (reference default)", "workers": f"0 -> {threads} hardware threads",
                   "corpus_builder": "reference Vocabulary::build (oracle/ref_capi.cpp ref_synth_corpus)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": phys, "threads": threads, "kind": "reference",
                         "sample": sample + f"; median of {args.steps} epochs, RunReport.epochs[0].words_per_sec"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_config(fw, args, mode, local, seed=1, epochs=None, workers=None):
    return fw.TrainConfig(dim=args.dim, window=args.window, negatives=args.negatives,
                          epochs=epochs or max(1, args.steps), workers=workers or args.chunks, streams=args.streams,
                          batch_sentences=args.batch_sentences, subsample=1e-4, seed=seed, deterministic=0,
                          reuse_mode=mode, device=local, sampler=args.sampler,
                          l1_refresh_log2=args.l1_refresh_log2, k1_lanes=args.k1_lanes, hot_rows=args.hot_rows,
                          hot_merge=args.hot_merge)


def roofline(args, words, seconds, mode, prof):
    peak, peak_src = load_peaks()
    bpw = algorithmic_bytes_per_word(args.dim, args.negatives)
    achieved = words * bpw / seconds / 1e9
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": None, "peak_source": peak_src, "bytes_per_word": bpw,
         "units_per_launch": "trained words; achieved = words per step x bytes_per_word / step device time"}
    p = prof.get(mode) if args.workload == "text8" and args.dim == 128 and args.negatives == 5 else None
    if p:
        wps = words / seconds
        r["traffic"] = p["dram_bytes_per_word"] * words  # per step, from the ncu launch list of the same launches
        r["dram_bytes_per_word"] = p["dram_bytes_per_word"]
        r["l2"] = {"bytes_per_word": p["l2_bytes_per_word"], "achieved": p["l2_bytes_per_word"] * wps / 1e9,
                   "peak": prof.get("l2_peak_gbs"), "unit": "GB/s",
                   "frac": (p["l2_bytes_per_word"] * wps / 1e9 / prof["l2_peak_gbs"]) if prof.get("l2_peak_gbs") else None,
                   "peak_source": prof.get("l2_peak_source")}
        r["issue"] = {"warp_inst_per_word": p["inst_per_word"],
                      "achieved_inst_per_s": p["inst_per_word"] * wps,
                      "peak_inst_per_s": prof.get("issue_peak"),
                      "frac": (p["inst_per_word"] * wps / prof["issue_peak"]) if prof.get("issue_peak") else None}
        r["source"] = prof.get("source")
    return r


def device_leg(fw, args, corpus, mode, local, steps):
    """Device-resident epochs on one GPU; returns (words per step, seconds list, launches per step)."""
    cfg = make_config(fw, args, mode, local, epochs=max(1, steps))
    with fw.Trainer(cfg, corpus.counts) as t:
        plan = t.plan_epoch(corpus, 0)
        for _ in range(args.warmup):
            plan.run()
        secs = [plan.run()[0] for _ in range(steps)]
        words, launches = plan.words, plan.batches + (2 if cfg.hot_rows > 0 else 0)
        plan.close()
    return words, secs, launches


def e2e_leg(fw, args, corpus, mode, local, steps):
    """One fw2v_train_corpus call of K epochs (one step = one epoch: every epoch is
    re-batched on the host, shipped H2D and trained; the pass counters come back
    D2H), timed around the whole call after a warm-up call."""
    epochs = max(1, min(steps, 20))
    cfg = make_config(fw, args, mode, local, epochs=epochs)
    with fw.Trainer(cfg, corpus.counts) as et:
        et.train_corpus(corpus)  # warm-up call (allocates pinned buffers)
        t0 = time.perf_counter()
        rep = et.train_corpus(corpus)
        secs = time.perf_counter() - t0
    return {"value": rep.words_trained / secs, "unit": UNIT, "h2d_bytes_per_step": int(rep.h2d_bytes // epochs),
            "d2h_bytes_per_step": 64 * args.streams, "epochs_per_call": epochs,
            "path": "fw2v_train_corpus (C-ABI), one call of K epochs: host batching threads -> pinned -> H2D -> "
                    "K1s, next epoch's first sub-batches shipped during this epoch's tail",
            "host_batching_words_per_sec_per_thread": rep.batching_words_per_sec, "batching_threads": args.streams}


def configs_leg(fw, args, corpus, local):
    """BASELINE.json configs[1] and [2] beside the headline: text8 at d=300 and the
    1bw-shaped corpus (534 M trained words per epoch) at d=128, both update orders,
    device-resident epochs on this GPU (the sweep, configs[4]: DESIGN.md section 6)."""
    import copy

    out = {}
    d300 = copy.copy(args)
    d300.dim = 300
    for mode in ("window_snapshot", "lifetime"):
        w, secs, _ = device_leg(fw, d300, corpus, mode, local, 5)
        out[f"text8_d300_{mode}"] = {"value": w * 5 / sum(secs), "unit": UNIT, "words_per_step": w}
    onebw = fw.synth_zipf(**fw.ONEBW_SHAPE)
    for mode in ("window_snapshot", "lifetime"):
        b = copy.copy(args)
        b.workload = "1bw"
        w, secs, _ = device_leg(fw, b, onebw, mode, local, 2)
        out[f"1bw_d128_{mode}"] = {"value": w * 2 / sum(secs), "unit": UNIT, "words_per_step": w,
                                   "roofline_frac": w * 2 / sum(secs) * algorithmic_bytes_per_word(128, args.negatives)
                                   / 1e9 / load_peaks()[0]}
    return out


def dropin_leg(fw, args, corpus):
    """Whole ringvec::train calls through the C++ drop-in, reference default
    TrainConfig (workers = 0 -> hardware threads) except the bench's shape."""
    try:
        h = fw.DropinHarness(corpus)
    except ImportError as e:
        return {"unavailable": str(e)}
    out = {"path": "ringvec::train (C++ drop-in, libringvec_fw2v.so) per call: fw2v_create (tables, HBM model, "
                   "init_model), host batching, H2D, kernels, model readback; reference default TrainConfig "
                   "(epochs=20, workers=0 -> hardware threads; drop-in defaults: alias sampler, top-64 hot-row "
                   "replicas with the live merge, auto in-flight budget)"}
    try:
        # drop-in defaults; then without the hot-row replicas (plain Hogwild on every row)
        for key, env in (("", {}), ("_no_hot_rows", {"FW2V_HOT_ROWS": "0"})):
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                for mode in ("lifetime", "window_snapshot"):
                    cfg = fw.TrainConfig(dim=args.dim, window=args.window, negatives=args.negatives, epochs=20,
                                         workers=0, batch_sentences=args.batch_sentences, subsample=1e-4, seed=1,
                                         reuse_mode=mode)
                    h.train(cfg)  # warm-up (first CUDA context, page-in, buffer cache)
                    calls = [h.train(cfg) for _ in range(3)]
                    best = sorted(calls, key=lambda r: r.call_seconds)[1]
                    out[mode + key] = {"value": best.words_trained / best.call_seconds, "unit": UNIT,
                                       "call_seconds": best.call_seconds,
                                       "epoch_words_per_sec": best.epoch_words_per_sec, "words": best.words_trained}
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
    finally:
        h.close()
    return out


def run_single(args, local):
    import numpy as np  # noqa: F401

    import paper_2312_07743_b200 as fw

    shape = shape_of(args.workload)
    corpus = fw.synth_zipf(**shape)
    prof = load_profile()
    mode = args.reuse_mode
    # Headline leg, with the clocks sampled over its timed region.
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        words, secs, launches = device_leg(fw, args, corpus, mode, local, args.steps)
        wall = time.perf_counter() - t0
    t_dev = float(sum(secs))
    value = words * args.steps / t_dev
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": config_block(args, shape, words, 1, "single GPU"),
        "roofline": roofline(args, words, t_dev / args.steps, mode, prof),
        "gpu_launches": launches * args.steps, "clocks": clk.summary(), "wall_s_leg": wall,
    }
    if not args.no_e2e:
        line["e2e"] = e2e_leg(fw, args, corpus, mode, local, args.steps)
    if not args.no_lifetime and mode != "lifetime":
        lsteps = min(args.steps, 20)
        lw, lsecs, _ = device_leg(fw, args, corpus, "lifetime", local, lsteps)
        lt = float(sum(lsecs))
        lf = {"value": lw * lsteps / lt, "unit": UNIT, "ms_per_step": 1e3 * lt / lsteps, "steps": lsteps,
              "roofline": roofline(args, lw, lt / lsteps, "lifetime", prof),
              "note": "reference default update order (ReuseMode::lifetime, sweep_samples trainer.cpp:133-154): "
                      "K1s window staircase (anti-diagonal wavefronts of consecutive windows overlapped, "
                      "csrc/fw2v_stair.cuh)"}
        if not args.no_e2e:
            lf["e2e"] = e2e_leg(fw, args, corpus, "lifetime", local, lsteps)
        line["lifetime"] = lf
    if not args.no_dropin:
        line["dropin_e2e"] = dropin_leg(fw, args, corpus)
    if not args.no_configs and args.workload == "text8" and args.dim == 128:
        line["other_configs"] = configs_leg(fw, args, corpus, local)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(args)
    print(json.dumps(line), flush=True)


def config_block(args, shape, words, world, parallelism):
    return {"workload": f"{args.workload}-shaped Zipf corpus ({shape['types']} ranks, "
                        f"{shape['tokens']} tokens, 1000-token sentences), 1 epoch per step",
            "dim": args.dim, "window": args.window, "negatives": args.negatives, "subsample": 1e-4,
            "words_per_step_per_gpu": words, "batch_sentences": args.batch_sentences,
            "streams": args.streams, "chunks": args.chunks, "reuse_mode": args.reuse_mode,
            "kernel": ("K1s (FULL-W2V independent negatives, Hogwild)" if args.reuse_mode == "window_snapshot"
                       else "K1s window staircase (reference lifetime order, Hogwild)"), "sampler": args.sampler,
            "l1_refresh_log2": args.l1_refresh_log2,
            "deviations": {"hot_rows": (f"top {args.hot_rows} output rows trained as 16 replicas merged live (every "
                                        "replica's updates summed into the others every few microseconds by a resident "
                                        "merge block: plain Hogwild's step, tests/test_hot_live.py)" if args.hot_merge
                                        else f"top {args.hot_rows} output rows trained as 16 replicas merged as their mean "
                                        "after each pass (1/16 of plain Hogwild's step)") if args.hot_rows else "off",
                           "l1_staging": (f"window-snapshot order: sample rows staged through L1, refreshed every "
                                          f"2^{args.l1_refresh_log2} windows per SM (other sentences' updates seen up to "
                                          "that late); lifetime order stages through L2 only (cp.async.cg): no staleness "
                                          "beyond Hogwild's in-flight updates"),
                           "sigmoid": "tanh.approx (|err| < 1e-3, SPEC.md:252)"},
            "parallelism": parallelism,
            "l2_policy": "inputs (238 MB id/negative stream per step) > 126 MB L2; no flush"}


def run_multi(args, world, rank, local, dist, shared):
    """One process per GPU: replica per rank, contiguous shard of whole chunks,
    merges inside the timed region (library NCCL; gloo exchange when ranks share
    a GPU)."""
    import numpy as np
    import torch

    import paper_2312_07743_b200 as fw
    from paper_2312_07743_b200.dist import TorchExchange, dp_chunks

    if args.workload == "text8":  # weak scaling: world x text8 tokens, one text8-sized shard per GPU
        shape = dict(types=TEXT8["types"], tokens=TEXT8["tokens"] * world)
        scaling = "weak"
    else:  # strong scaling: the 1bw-shaped corpus split across the ranks
        shape = ONEBW
        scaling = "strong"
    corpus = fw.synth_zipf(**shape)
    mode = args.reuse_mode
    cfg = make_config(fw, args, mode, local, epochs=max(1, args.steps))
    t = fw.Trainer(cfg, corpus.counts)
    exchange = None
    if shared:
        exchange = TorchExchange()
    else:
        obj = [fw.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        t.comm_init_rank(obj[0], world, rank)
    # The partition fw2v_train_corpus_multi uses: whole chunks per shard and round.
    est_words = 0.592 * shape["tokens"] / world  # trained words per shard (subsample 1e-4 keeps ~59%)
    rounds = max(1, round(est_words / args.average_words)) if args.average_words > 0 else 1
    total, per_shard, per_round = dp_chunks(args.chunks, world, rounds)
    plans = [t.plan_chunks(corpus, total, rank * per_shard + r * per_round, rank * per_shard + (r + 1) * per_round,
                           words_base=0, words_scale=world) for r in range(rounds)]
    words = sum(p.words for p in plans)
    fw.merge_begin([t])

    def step():
        dev, merge = 0.0, 0.0
        for p in plans:
            s, _ = p.run()
            dev += s
            m0 = time.perf_counter()
            fw.merge_replicas([t], [p.words], n_shards=world, exchange=exchange)
            merge += time.perf_counter() - m0
        return dev, merge

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    dev_t, merge_t = 0.0, 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            a, b = step()
            dev_t += a
            merge_t += b
    dist.barrier()
    tt = torch.tensor([dev_t + merge_t, merge_t], dtype=torch.float64)
    if not shared:
        tt = tt.cuda()
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max, merge_max = float(tt[0].item()), float(tt[1].item())
    total_words = torch.tensor([words * args.steps], dtype=torch.float64)
    if not shared:
        total_words = total_words.cuda()
    dist.all_reduce(total_words)
    value = float(total_words.item()) / t_max
    for p in plans:
        p.close()
    e2e = None
    if not args.no_e2e:
        et = fw.Trainer(make_config(fw, args, mode, local, epochs=1), corpus.counts)
        if not shared:
            obj = [fw.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            et.comm_init_rank(obj[0], world, rank)
        fw.train_corpus_multi([et], corpus, average_words=args.average_words, shard0=rank, n_shards=world,
                              exchange=exchange)  # warm-up
        ew, es = 0, 0.0
        for _ in range(max(1, min(args.steps, 3))):
            dist.barrier()
            rep = fw.train_corpus_multi([et], corpus, average_words=args.average_words, shard0=rank,
                                        n_shards=world, exchange=exchange)
            ew += rep.words_trained
            es += rep.wall_seconds
            h2d = rep.h2d_bytes
        te = torch.tensor([es], dtype=torch.float64)
        tw = torch.tensor([ew], dtype=torch.float64)
        if not shared:
            te, tw = te.cuda(), tw.cuda()
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dist.all_reduce(tw)
        e2e = {"value": float(tw.item()) / float(te.item()), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 64 * args.streams,
               "path": "fw2v_train_corpus_multi (C-ABI) per rank: shard batching -> H2D -> K1s, merges via NCCL"}
        et.close()
    if rank == 0:
        prof = load_profile()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": config_block(args, shape, words, world,
                                   f"dp{world}: replica per GPU, contiguous shard, {rounds} merge(s) per step "
                                   f"({cfg.replica_merge} rule) via NCCL all-reduce, inside the timed region"),
            "roofline": roofline(args, words, t_max / args.steps, mode, prof),
            "merge_ms_per_step": 1e3 * merge_max / args.steps,
            "e2e": e2e, "gpu_launches": (sum(p.batches for p in plans) + 4 * rounds) * args.steps,
            "clocks": clk.summary(),
        }
        if shared:
            line["note"] = "ranks share GPUs (gloo exchange): functional check, not a measurement"
        print(json.dumps(line), flush=True)
    t.close()


def cpu_baseline_leg(args):
    from oracle.oracle import Oracle, RefCorpus, TrainConfig as RConfig, available

    kind = "reference" if available("ref") else "port"
    phys, threads = host_cores()
    if kind == "port":  # the C restatement (workers = 1 only)
        import paper_2312_07743_b200 as fw

        c = fw.synth_zipf(**shape_of(args.workload)).head(300)
        o = Oracle("oracle")
        cfg = RConfig(dim=args.dim, window=args.window, negatives=args.negatives, epochs=1, workers=1,
                      batch_sentences=args.batch_sentences, subsample=1e-4, seed=1)
        _, _, rep = o.train(c.counts, c.offsets, c.ids, cfg)
        return {"value": rep.epoch_words_per_sec[0], "unit": UNIT, "cores": 1, "kind": kind,
                "sample": "first 300 sentences, 1 epoch, oracle port, workers=1"}
    ref = Oracle("ref")
    shape = shape_of(args.workload)
    n = 4000
    corpus = RefCorpus(ref, shape["types"], shape["tokens"]).head(n)
    cfg = RConfig(dim=args.dim, window=args.window, negatives=args.negatives, epochs=1, workers=0,
                  batch_sentences=args.batch_sentences, subsample=1e-4, seed=1)
    rep = corpus.train(cfg)
    return {"value": rep.epoch_words_per_sec[0], "unit": UNIT, "cores": phys, "threads": threads, "kind": kind,
            "sample": f"first {n} sentences of the {args.workload}-shaped corpus (reference Vocabulary::build), "
                      f"1 epoch, reference lifetime mode, workers=0 -> {threads} threads"}


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
    ap.add_argument("--hot-rows", type=int, default=64)
    ap.add_argument("--hot-merge", type=int, default=1, help="1 live sum merge of the hot-row replicas, 0 pass-end mean")
    ap.add_argument("--average-words", type=int, default=25_000_000,
                    help="multi-GPU: merge the replicas every this many trained words per GPU")
    ap.add_argument("--ref-budget-s", type=float, default=200.0,
                    help="--impl reference: wall budget of the whole run (sizes the per-step sample)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-lifetime", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the text8 d=300 and 1bw legs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, local, dist, shared = dist_setup()
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        elif world == 1:
            run_single(args, local)
        else:
            run_multi(args, world, rank, local, dist, shared)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
