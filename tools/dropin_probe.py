"""Why is the ringvec::train drop-in slow with reference defaults? Times whole
drop-in calls (DropinHarness) under FW2V_* variants, and the same config through
fw2v_train_corpus. usage: python tools/dropin_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402

corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
print("hardware threads", os.cpu_count(), flush=True)
VARIANTS = [
    {},
    {"FW2V_MAX_INFLIGHT": "-1"},
    {"FW2V_HOT_ROWS": "64"},
    {"FW2V_HOT_ROWS": "64", "FW2V_MAX_INFLIGHT": "-1"},
    {"FW2V_STREAMS": "16"},
]
for mode in ("lifetime", "window_snapshot"):
    for var in VARIANTS:
        for k, v in var.items():
            os.environ[k] = v
        cfg = fw.TrainConfig(dim=128, window=5, negatives=5, epochs=1, workers=0, batch_sentences=10000,
                             subsample=1e-4, seed=1, reuse_mode=mode)
        h = fw.DropinHarness(corpus)
        try:
            h.train(cfg)
            r = h.train(cfg)
            print(f"dropin {mode:16s} {var}: call {r.call_seconds:.3f} s, {r.words_trained / r.call_seconds / 1e6:.1f} "
                  f"Mw/s (epoch {r.epoch_words_per_sec / 1e6:.1f} Mw/s)", flush=True)
        finally:
            h.close()
        for k in var:
            del os.environ[k]
    for hot, mi in ((0, 0), (0, -1), (64, 0)):
        cfg = fw.TrainConfig(dim=128, window=5, negatives=5, epochs=1, workers=0, batch_sentences=10000,
                             subsample=1e-4, seed=1, reuse_mode=mode, sampler="alias", hot_rows=hot, max_inflight=mi,
                             deterministic=0)
        with fw.Trainer(cfg, corpus.counts) as t:
            t.train_corpus(corpus)
            t0 = time.perf_counter()
            rep = t.train_corpus(corpus)
            dt = time.perf_counter() - t0
        print(f"train_corpus {mode:16s} hot {hot} max_inflight {mi}: {rep.words_trained / dt / 1e6:.1f} Mw/s "
              f"kernel {rep.kernel_seconds:.4f} s", flush=True)
