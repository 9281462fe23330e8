"""Golden digests of the reference trainer at the BASELINE text8 shape.

Runs the REFERENCE ``ringvec::train`` (oracle/_ref, compiled from
/root/reference/proj by oracle/Makefile) with ``workers = 1`` — the
reference's fully deterministic mode (trainer.hpp:115-118, trainer.cpp:390-528)
— for ONE epoch on the text8-shaped synthetic corpus (BASELINE.json
configs[0] / configs[1]; corpus from ``fw2v_corpus_synth_zipf``, which is
deterministic) at d=128 and d=300, and records SHA-256 digests of both
embedding matrices plus counters. The 73 / 171 MB matrices do not fit in the
repo; the digests do, and tests/test_gpu_parity.py::test_text8_k2_equals_reference
compares the GPU's deterministic engine (K2) against them on the B200 box,
where /root/reference does not exist.

Run here (needs oracle/_ref and libfw2v.so built; ~2 + ~5 min of one core):
    python tests/golden/make_text8_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "tests", "golden", "text8_ref_workers1.json")

# Reference TrainConfig (config.hpp:13-35) with the bench's text8 settings.
BASE = dict(window=5, negatives=5, epochs=1, workers=1, batch_sentences=10000, subsample=1e-4, seed=1,
            alpha0=0.025, table_size=10_000_000, table_power=0.75)


def corpus_digest(c) -> str:
    h = hashlib.sha256()
    for a in (c.counts, c.offsets, c.ids):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def matrix_digest(m: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(m, dtype="<f4").tobytes()).hexdigest()


def main(dims=(128, 300)):
    import paper_2312_07743_b200 as fw
    from oracle.oracle import Oracle, TrainConfig

    corpus = fw.synth_zipf(**fw.TEXT8_SHAPE)
    ref = Oracle("ref")
    out = {"generator": "tests/golden/make_text8_golden.py (reference ringvec::train, oracle/_ref, workers=1)",
           "corpus": {"shape": fw.TEXT8_SHAPE, "sha256": corpus_digest(corpus),
                      "sentences": int(len(corpus.offsets) - 1), "tokens": int(corpus.offsets[-1]),
                      "vocab": int(len(corpus.counts))},
           "config": BASE, "runs": {}}
    if os.path.exists(OUT):
        with open(OUT) as f:
            prev = json.load(f)
        if prev.get("corpus", {}).get("sha256") == out["corpus"]["sha256"]:
            out["runs"] = prev.get("runs", {})
    for d in dims:
        t0 = time.time()
        cfg = TrainConfig(dim=d, **BASE)
        inp, outp, rep = ref.train(corpus.counts, corpus.offsets, corpus.ids, cfg)
        secs = time.time() - t0
        out["runs"][str(d)] = {
            "input_sha256": matrix_digest(inp), "output_sha256": matrix_digest(outp),
            "words_trained": int(rep.words_trained), "sentences_trained": int(rep.sentences_trained),
            "traffic": [int(x) for x in rep.traffic],
            "input_fro": float(np.linalg.norm(inp.astype(np.float64))),
            "output_fro": float(np.linalg.norm(outp.astype(np.float64))),
            "input_row1_head": [float(x) for x in inp[1, :8]],
            "output_row1_head": [float(x) for x in outp[1, :8]],
            "reference_seconds_1_thread": round(secs, 1),
        }
        print(d, out["runs"][str(d)], flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(tuple(int(x) for x in sys.argv[1:]) or (128, 300))
