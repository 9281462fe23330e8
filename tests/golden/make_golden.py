"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, compiled
from /root/reference/proj by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the C oracle (tests/test_oracle.py) on machines where the
reference sources are absent (the GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
from helpers import fixed_negatives, random_corpus  # noqa: E402
from oracle.oracle import Oracle, TrainConfig  # noqa: E402

TRAIN_CASES = {
    # name: (corpus args, config)
    "train_d12_w5_n5_sub": ((40, 20, 30, 11), dict(dim=12, window=5, negatives=5, epochs=2, workers=1,
                                                   batch_sentences=7, table_size=4001, subsample=1e-2, seed=42)),
    "train_d16_w7_n3": ((30, 25, 20, 12), dict(dim=16, window=7, negatives=3, epochs=1, workers=1,
                                              batch_sentences=5, table_size=997, subsample=0.0, seed=7)),
    "train_d8_w2_n0": ((25, 15, 12, 13), dict(dim=8, window=2, negatives=0, epochs=2, workers=1,
                                             batch_sentences=4, table_size=100, subsample=0.0, seed=3)),
}
SENT_CASES = {
    # train_sentence sequences with fixed negatives/alphas for each reuse mode
    f"sent_{mode}": (mode, (8, 18, 14, 21)) for mode in ["lifetime", "window", "none", "window_snapshot"]
}


def main():
    ref = Oracle("ref")
    for name, (cargs, cfg) in TRAIN_CASES.items():
        counts, offsets, ids = random_corpus(*cargs)
        inp, out, rep = ref.train(counts, offsets, ids, TrainConfig(**cfg))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), counts=counts, offsets=offsets, ids=ids,
                            input=inp, output=out, words=rep.words_trained, traffic=np.array(rep.traffic),
                            epoch_words=np.array(rep.epoch_words), cfg=repr(cfg))
    for name, (mode, cargs) in SENT_CASES.items():
        counts, offsets, ids = random_corpus(*cargs)
        v = len(counts)
        negs = fixed_negatives(int(offsets[-1]), 5, v, 17)
        alphas = np.linspace(0.03, 0.01, len(offsets) - 1).astype(np.float32)
        inp, _ = ref.init_model(v, 10, 99)
        out = (inp[::-1] * 2.0).copy()
        inp0, out0 = inp.copy(), out.copy()
        ctr = ref.train_sentences(inp, out, offsets, ids, negs, alphas,
                                  TrainConfig(dim=10, window=5, negatives=5, reuse_mode=mode))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), counts=counts, offsets=offsets, ids=ids, negs=negs,
                            alphas=alphas, input0=inp0, output0=out0, input=inp, output=out,
                            counters=np.array(ctr), mode=mode)
    # scalar golden values straight from the reference
    xs = np.array([-100.0, -6.0, -3.3, -0.7, 0.0, 0.25, 1.0, 5.9, 6.0, 1000.0], np.float32)
    sig = np.array([ref.sigmoid(float(x)) for x in xs], np.float32)
    lr = np.array([ref.lr_at(w, 1000, 0.025) for w in [0, 1, 500, 999, 1000, 5000]], np.float32)
    draws = ref.rng_draws(1, 2, 3, 4, 64)
    init_i, _ = ref.init_model(7, 5, 123)
    counts = np.array([16, 9, 9, 5, 1], np.uint64)
    tab = ref.table(counts, 0.75, 101)
    keep = ref.keep_probs(np.array([1000, 100, 10, 1], np.uint64), 1e-2)
    np.savez_compressed(os.path.join(HERE, "scalars.npz"), sig_x=xs, sig=sig, lr=lr, draws=draws, init=init_i,
                        table=tab, keep=keep)
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
