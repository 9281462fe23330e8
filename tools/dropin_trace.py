"""FW2V_TRACE timelines of one drop-in call and one fw2v_train_corpus call with
the same configuration (diagnostics). usage: python tools/dropin_trace.py [dropin|corpus]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402

corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
cfg = fw.TrainConfig(dim=128, window=5, negatives=5, epochs=1, workers=0, batch_sentences=10000, subsample=1e-4,
                     seed=1, reuse_mode="window_snapshot", sampler="alias", hot_rows=0, deterministic=0)
if sys.argv[1] == "dropin":
    h = fw.DropinHarness(corpus)
    h.train(cfg)
    r = h.train(cfg)
    print("dropin call", r.call_seconds, "epoch w/s", r.epoch_words_per_sec, flush=True)
else:
    with fw.Trainer(cfg, corpus.counts) as t:
        t.train_corpus(corpus)
        rep = t.train_corpus(corpus)
    print("corpus", rep.wall_seconds, rep.words_trained / rep.wall_seconds, flush=True)
