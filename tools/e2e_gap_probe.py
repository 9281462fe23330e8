"""Where does the e2e epoch (fw2v_train_corpus, bench config) lose against the
device-resident plan? Prints wall vs kernel span per epoch and the FW2V_TRACE
timeline summary (first kernel start, last kernel end, busy union).
usage: FW2V_TRACE=1 python tools/e2e_gap_probe.py 2> trace.txt"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402

corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
cfg = fw.TrainConfig(dim=128, window=5, negatives=5, epochs=1, workers=64, streams=16, batch_sentences=10000,
                     subsample=1e-4, seed=1, deterministic=0, reuse_mode="window_snapshot", sampler="alias",
                     l1_refresh_log2=5, hot_rows=64)
with fw.Trainer(cfg, corpus.counts) as t:
    for it in range(4):
        t0 = time.perf_counter()
        rep = t.train_corpus(corpus)
        dt = time.perf_counter() - t0
        print(f"epoch {it}: wall {dt * 1e3:.2f} ms, report wall {rep.wall_seconds * 1e3:.2f} ms, kernel span "
              f"{rep.kernel_seconds * 1e3:.2f} ms, {rep.words_trained / dt / 1e6:.1f} Mw/s, batching "
              f"{rep.batching_words_per_sec / 1e6:.1f} Mw/s/thread", flush=True)
    import dataclasses
    with fw.Trainer(dataclasses.replace(cfg, epochs=10), corpus.counts) as t10:
        t10.train_corpus(corpus)
        t0 = time.perf_counter()
        rep = t10.train_corpus(corpus)
        dt = time.perf_counter() - t0
        print(f"10-epoch call: {dt * 1e3 / 10:.2f} ms/epoch, {rep.words_trained / dt / 1e6:.1f} Mw/s", flush=True)
    plan = t.plan_epoch(corpus, 0)
    for it in range(3):
        s, _ = plan.run()
        print(f"plan: {s * 1e3:.2f} ms, {plan.words / s / 1e6:.1f} Mw/s", flush=True)
    plan.close()
