"""ctypes bindings for the CPU checkers — TEST INFRASTRUCTURE, never the product.

Two checkers with one Python surface:

* ``Oracle("oracle")``: the plain-C restatement ``oracle/lib/libfw2v_oracle.so``
  (oracle/fw2v_oracle.c; every function cites the reference file:line it restates).
* ``Oracle("ref")``: the reference itself, compiled from /root/reference/proj by
  oracle/Makefile into ``oracle/_ref/libringvec_refcapi.so`` (oracle/ref_capi.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "oracle": os.path.join(HERE, "lib", "libfw2v_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libringvec_refcapi.so"),
}

REUSE_MODES = {"lifetime": 0, "window": 1, "none": 2, "window_snapshot": 3}


class CConfig(C.Structure):
    """Field-for-field mirror of ringvec::TrainConfig (config.hpp:13-35)."""

    _fields_ = [
        ("dim", C.c_int32), ("window", C.c_int32), ("negatives", C.c_int32), ("epochs", C.c_int32),
        ("alpha0", C.c_float), ("subsample", C.c_double),
        ("min_count", C.c_uint64), ("batch_sentences", C.c_uint64), ("max_sentence_len", C.c_uint64),
        ("workers", C.c_int32), ("seed", C.c_uint64), ("reuse_mode", C.c_int32),
        ("table_power", C.c_double), ("table_size", C.c_uint64), ("queue_capacity", C.c_uint64),
        ("ignore_delimiters", C.c_int32),
    ]


class CReport(C.Structure):
    _fields_ = [
        ("words_trained", C.c_uint64), ("sentences_trained", C.c_uint64), ("vocab_size", C.c_uint64),
        ("wall_seconds", C.c_double), ("batching_words_per_sec", C.c_double),
        ("n_epochs", C.c_int32),
        ("epoch_words", C.c_uint64 * 64), ("epoch_seconds", C.c_double * 64),
        ("epoch_words_per_sec", C.c_double * 64),
        ("traffic", C.c_uint64 * 5), ("analytic", C.c_uint64 * 5),
    ]


@dataclass
class TrainConfig:
    """Python mirror of ringvec::TrainConfig defaults (config.hpp:13-35)."""

    dim: int = 128
    window: int = 5
    negatives: int = 5
    epochs: int = 20
    alpha0: float = 0.025
    subsample: float = 1e-4
    min_count: int = 5
    batch_sentences: int = 10000
    max_sentence_len: int = 1000
    workers: int = 0
    seed: int = 1
    reuse_mode: str = "lifetime"
    table_power: float = 0.75
    table_size: int = 10_000_000
    queue_capacity: int = 0
    ignore_delimiters: bool = True

    @property
    def context_width(self) -> int:
        return (self.window + 1) // 2

    def to_c(self) -> CConfig:
        c = CConfig()
        for name, _ in CConfig._fields_:
            v = getattr(self, name)
            if name == "reuse_mode":
                v = REUSE_MODES[v]
            elif name == "ignore_delimiters":
                v = int(bool(v))
            setattr(c, name, v)
        return c


@dataclass
class Report:
    words_trained: int
    sentences_trained: int
    wall_seconds: float
    batching_words_per_sec: float
    epoch_words: list = field(default_factory=list)
    epoch_words_per_sec: list = field(default_factory=list)
    traffic: tuple = ()
    analytic: tuple = ()

    @staticmethod
    def from_c(r: CReport) -> "Report":
        n = r.n_epochs
        return Report(r.words_trained, r.sentences_trained, r.wall_seconds, r.batching_words_per_sec,
                      list(r.epoch_words[:n]), list(r.epoch_words_per_sec[:n]),
                      tuple(r.traffic), tuple(r.analytic))


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Oracle:
    def __init__(self, kind: str = "oracle"):
        path = LIB_PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        self.kind = kind
        self.lib = C.CDLL(path)
        pre = "oracle_" if kind == "oracle" else "ref_"
        self._pre = pre
        L = self.lib
        f = lambda n: getattr(L, pre + n)  # noqa: E731
        f("last_error").restype = C.c_char_p
        f("sigmoid").restype = C.c_float
        f("sigmoid").argtypes = [C.c_float]
        f("lr_at").restype = C.c_float
        f("lr_at").argtypes = [C.c_uint64, C.c_uint64, C.c_float]
        f("assemble_batch").restype = C.c_int64

    def _fn(self, name):
        return getattr(self.lib, self._pre + name)

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"{self.kind}: error {rc}: {self._fn('last_error')().decode()}")

    def save_embeddings(self, path, rows, counts, which=0):
        """Reference save_embeddings with the ref_capi token names (w%09d); ref only."""
        rows = np.ascontiguousarray(rows, np.float32)
        counts = np.ascontiguousarray(counts, np.uint64)
        self._check(self._fn("save_embeddings")(counts.ctypes.data_as(C.POINTER(C.c_uint64)), rows.shape[0],
                                                rows.shape[1], rows.ctypes.data_as(C.POINTER(C.c_float)), which,
                                                os.fsencode(str(path))))

    def nearest_neighbors(self, rows, queries, k):
        """Reference nearest_neighbors per query id -> (ids, cos), ref only."""
        rows = np.ascontiguousarray(rows, np.float32)
        q = np.ascontiguousarray(queries, np.int32)
        ids = np.zeros((len(q), k), np.int32)
        cos = np.zeros((len(q), k), np.float64)
        self._check(self._fn("nearest_neighbors")(rows.ctypes.data_as(C.POINTER(C.c_float)), rows.shape[0],
                                                  rows.shape[1], q.ctypes.data_as(C.POINTER(C.c_int32)), len(q), k,
                                                  ids.ctypes.data_as(C.POINTER(C.c_int32)),
                                                  cos.ctypes.data_as(C.POINTER(C.c_double))))
        return ids, cos

    def analogy_correct(self, rows, quads, method):
        """Reference eval_analogy on each quadruple alone: 1 where it predicts quads[:, 3]."""
        rows = np.ascontiguousarray(rows, np.float32)
        qd = np.ascontiguousarray(quads, np.int32)
        out = np.zeros(len(qd), np.int32)
        self._check(self._fn("analogy_correct")(rows.ctypes.data_as(C.POINTER(C.c_float)), rows.shape[0],
                                                rows.shape[1], qd.ctypes.data_as(C.POINTER(C.c_int32)), len(qd),
                                                method, out.ctypes.data_as(C.POINTER(C.c_int32))))
        return out

    # -- scalar helpers ------------------------------------------------------
    def sigmoid(self, x: float) -> float:
        return self._fn("sigmoid")(x)

    def lr_at(self, trained: int, total: int, alpha0: float) -> float:
        return self._fn("lr_at")(trained, total, alpha0)

    def rng_draws(self, seed, a, b, c, n) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._fn("rng_draws")(C.c_uint64(seed), C.c_uint64(a), C.c_uint64(b), C.c_uint64(c),
                              C.c_uint64(n), _p(out, C.c_uint64))
        return out

    def init_model(self, vocab: int, dim: int, seed: int):
        n = vocab * dim
        i = np.zeros(n, np.float32)
        o = np.ones(n, np.float32)
        self._check(self._fn("init_model")(vocab, dim, C.c_uint64(seed), _p(i, C.c_float), _p(o, C.c_float)))
        return i.reshape(vocab, dim), o.reshape(vocab, dim)

    def keep_probs(self, counts: np.ndarray, threshold: float):
        counts = np.ascontiguousarray(counts, np.uint64)
        out = np.zeros(len(counts), np.float64)
        rc = self._fn("keep_probs")(_p(counts, C.c_uint64), len(counts), C.c_double(threshold),
                                   _p(out, C.c_double))
        if rc < 0:
            self._check(-rc)
        return out if rc == 1 else None

    def table(self, counts: np.ndarray, power: float, size: int) -> np.ndarray:
        counts = np.ascontiguousarray(counts, np.uint64)
        out = np.zeros(size, np.int32)
        self._check(self._fn("table_build")(_p(counts, C.c_uint64), len(counts), C.c_double(power),
                                            C.c_uint64(size), _p(out, C.c_int32)))
        return out

    def assemble_batch(self, counts, offsets, ids, cursor, max_sentences, negatives, power,
                       table_size, threshold, seed, a, b, c):
        counts = np.ascontiguousarray(counts, np.uint64)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        ids = np.ascontiguousarray(ids, np.int32)
        cap = len(ids) + 1
        o_ids = np.zeros(cap, np.int32)
        o_off = np.zeros(len(offsets) + 1, np.uint64)
        o_negs = np.zeros(cap * max(negatives, 1), np.int32)
        cur = C.c_uint64(cursor)
        n = self._fn("assemble_batch")(
            _p(counts, C.c_uint64), len(counts), _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1),
            _p(ids, C.c_int32), C.byref(cur), C.c_uint64(max_sentences), negatives, C.c_double(power),
            C.c_uint64(table_size), C.c_double(threshold), C.c_uint64(seed), C.c_uint64(a),
            C.c_uint64(b), C.c_uint64(c), _p(o_ids, C.c_int32), _p(o_off, C.c_uint64),
            _p(o_negs, C.c_int32))
        if n < 0:
            self._check(-n)
        off = o_off[: n + 1].copy()
        w = int(off[-1])
        return cur.value, off, o_ids[:w].copy(), o_negs[: w * negatives].copy()

    def analytic_traffic(self, length, width, negatives, mode="lifetime"):
        out = np.zeros(5, np.uint64)
        self._check(self._fn("analytic_traffic")(C.c_uint64(length), width, negatives,
                                                 REUSE_MODES[mode], _p(out, C.c_uint64)))
        return tuple(int(x) for x in out)

    # -- training --------------------------------------------------------------
    def train_sentences(self, inp, out, offsets, ids, negatives, alphas, cfg: TrainConfig):
        """Serial train_sentence (trainer.cpp:332) over sentences; updates inp/out in place."""
        assert inp.dtype == np.float32 and inp.flags.c_contiguous and out.flags.c_contiguous
        v, d = inp.shape
        offsets = np.ascontiguousarray(offsets, np.uint64)
        ids = np.ascontiguousarray(ids, np.int32)
        negatives = np.ascontiguousarray(negatives, np.int32)
        if negatives.size == 0:
            negatives = np.zeros(1, np.int32)
        alphas = np.ascontiguousarray(alphas, np.float32)
        counters = np.zeros(5, np.uint64)
        c = cfg.to_c()
        self._check(self._fn("train_sentences")(
            _p(inp, C.c_float), _p(out, C.c_float), v, d, _p(offsets, C.c_uint64),
            C.c_uint64(len(offsets) - 1), _p(ids, C.c_int32), _p(negatives, C.c_int32),
            _p(alphas, C.c_float), C.byref(c), _p(counters, C.c_uint64)))
        return tuple(int(x) for x in counters)

    def train(self, counts, offsets, ids, cfg: TrainConfig):
        """ringvec::train (trainer.cpp:390). The oracle restates workers = 1 only."""
        counts = np.ascontiguousarray(counts, np.uint64)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        ids = np.ascontiguousarray(ids, np.int32)
        v = len(counts)
        inp = np.zeros((v, cfg.dim), np.float32)
        out = np.zeros((v, cfg.dim), np.float32)
        rep = CReport()
        c = cfg.to_c()
        self._check(self._fn("train")(
            _p(counts, C.c_uint64), v, _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1),
            _p(ids, C.c_int32), C.byref(c), _p(inp, C.c_float), _p(out, C.c_float), C.byref(rep)))
        return inp, out, Report.from_c(rep)


class RefCorpus:
    """A ringvec::Corpus built by the reference (ref_synth_corpus): the bench's
    reference arm trains it without loading libfw2v. ref only."""

    def __init__(self, oracle: "Oracle", types=0, tokens=0, s=1.0, sentence_len=1000, min_count=5, _handle=None):
        self.o = oracle
        h = _handle if _handle is not None else C.c_void_p()
        if _handle is None:
            oracle._check(oracle._fn("synth_corpus")(C.c_uint64(types), C.c_uint64(tokens), C.c_double(s),
                                                     C.c_uint64(sentence_len), C.c_uint64(min_count), C.byref(h)))
        self.h = h
        pc, v, ns, ni = C.POINTER(C.c_uint64)(), C.c_int32(), C.c_uint64(), C.c_uint64()
        oracle._fn("corpus_view")(h, C.byref(pc), C.byref(v), C.byref(ns), C.byref(ni))
        self.counts = np.ctypeslib.as_array(pc, (v.value,)).copy()
        self.n_sentences, self.n_ids = ns.value, ni.value

    def arrays(self):
        off = np.zeros(self.n_sentences + 1, np.uint64)
        ids = np.zeros(self.n_ids, np.int32)
        self.o._fn("corpus_export")(self.h, _p(off, C.c_uint64), _p(ids, C.c_int32))
        return off, ids

    def head(self, n_sentences: int) -> "RefCorpus":
        h = C.c_void_p()
        self.o._check(self.o._fn("corpus_head")(self.h, C.c_uint64(n_sentences), C.byref(h)))
        return RefCorpus(self.o, _handle=h)

    def train(self, cfg: TrainConfig) -> Report:
        rep = CReport()
        c = cfg.to_c()
        self.o._check(self.o._fn("train_corpus")(self.h, C.byref(c), C.byref(rep)))
        return Report.from_c(rep)

    def __del__(self):
        if getattr(self, "h", None):
            self.o._fn("corpus_free")(self.h)
            self.h = None


def available(kind: str) -> bool:
    return os.path.exists(LIB_PATHS[kind])
