"""Phases of a drop-in-equivalent call (reference default TrainConfig, 20 epochs,
workers = 0) through the Python binding: create, train_corpus, get_model, destroy;
then the whole ringvec::train call through the harness."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402

corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
for mode in ("window_snapshot", "lifetime"):
    for it in range(2):
        cfg = fw.TrainConfig(dim=128, window=5, negatives=5, epochs=20, workers=0, batch_sentences=10000,
                             subsample=1e-4, seed=1, reuse_mode=mode, sampler="alias", deterministic=0)
        t0 = time.perf_counter()
        t = fw.Trainer(cfg, corpus.counts)
        t1 = time.perf_counter()
        rep = t.train_corpus(corpus)
        t2 = time.perf_counter()
        t.get_model()
        t3 = time.perf_counter()
        t.close()
        t4 = time.perf_counter()
        eps = [e["seconds"] for e in rep.epochs]
        print(f"{mode} run {it}: create {1e3 * (t1 - t0):.1f} ms, train {1e3 * (t2 - t1):.1f} ms "
              f"({rep.words_trained / (t2 - t1) / 1e6:.0f} Mw/s; epochs {1e3 * min(eps):.2f}..{1e3 * max(eps):.2f} ms), "
              f"get_model {1e3 * (t3 - t2):.1f} ms, destroy {1e3 * (t4 - t3):.1f} ms", flush=True)
h = fw.DropinHarness(corpus)
for mode in ("window_snapshot", "lifetime"):
    cfg = fw.TrainConfig(dim=128, window=5, negatives=5, epochs=20, workers=0, batch_sentences=10000,
                         subsample=1e-4, seed=1, reuse_mode=mode)
    for it in range(3):
        r = h.train(cfg)
        print(f"harness {mode}: call {r.call_seconds * 1e3:.1f} ms, {r.words_trained / r.call_seconds / 1e6:.0f} Mw/s, "
              f"epoch rate {r.epoch_words_per_sec / 1e6:.0f}", flush=True)
h.close()
