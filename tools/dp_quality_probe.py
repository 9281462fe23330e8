"""Data-parallel merge-rule probe (one GPU, R replicas sharing it): SGNS loss of
R-replica runs vs the reference, per merge rule and averaging period.
usage: python tools/dp_quality_probe.py [planted|text8] R1,R2,.. rounds1,rounds2,..
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2312_07743_b200 as fw  # noqa: E402
from helpers import sgns_loss  # noqa: E402
from oracle.oracle import Oracle, TrainConfig as RConfig  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "planted"
Rs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
rounds_list = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,4").split(",")]
ref = Oracle("ref")
if which == "planted":
    from test_quality import CFG, _eval, planted_corpus

    counts, offsets, ids, word_topic = planted_corpus()
    base = dict(dim=64, **CFG)
    rin, rout, rrep = ref.train(counts, offsets, ids, RConfig(workers=16, **base))

    def ev(i, o):
        return _eval(i, o, offsets, ids, counts, word_topic)
    corpus = fw.Corpus(counts, offsets, ids)
else:
    corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
    counts = corpus.counts
    base = dict(dim=128, window=5, negatives=5, epochs=3, batch_sentences=10000, subsample=1e-4, seed=1)
    p = counts.astype(np.float64) ** 0.75
    negs = np.random.default_rng(5).choice(len(counts), 400_000 * 5, p=p / p.sum()).astype(np.int32)
    off = corpus.offsets[:401].copy()

    def ev(i, o):
        return sgns_loss(i, o, off, corpus.ids[: int(off[-1])], negs, wf=3, n_neg=5, max_pairs=100_000), 0.0
    rin, rout, rrep = ref.train(counts, corpus.offsets, corpus.ids, RConfig(workers=16, **base))
ref_loss, ref_rec = ev(rin, rout)
print(f"{which}: reference loss {ref_loss:.4f} recall {ref_rec:.4f} words {rrep.words_trained}", flush=True)
per_epoch = rrep.words_trained / base["epochs"]
for R in Rs:
    for rounds in rounds_list:
        for merge in ("mean", "touched"):
            cfg = fw.TrainConfig(workers=64, streams=16, deterministic=0, reuse_mode="window_snapshot",
                                 sampler="alias", replica_merge=merge, **base)
            ts = [fw.Trainer(cfg, counts) for _ in range(R)]
            try:
                rep = fw.train_corpus_multi(ts, corpus, average_words=int(per_epoch / R / rounds))
                gi, go = ts[0].get_model()
            finally:
                for t in ts:
                    t.close()
            loss, rec = ev(gi, go)
            print(f"R={R} rounds/epoch={rounds} merge={merge:8s} loss {loss:.4f} ({100 * (loss / ref_loss - 1):+.2f}%) "
                  f"recall {rec:.4f} words {rep.words_trained} finite {np.isfinite(gi).all()}", flush=True)
