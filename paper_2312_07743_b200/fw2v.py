"""Python binding of the B200 FULL-W2V trainer C-ABI (include/fw2v.h).

Thin ctypes layer over ``_lib/libfw2v.so``; the product is the C++/CUDA
library, this module only marshals numpy arrays. There is no CPU training
path: if the shared library is missing, importing the trainer raises, and on a
machine without a CUDA device every training call fails with
``FW2V_ERR_NO_DEVICE``.

The surface mirrors the reference C++ API (``/root/reference/proj``):
``TrainConfig`` (config.hpp:13-35), ``Trainer.train_corpus`` ≈ ``ringvec::train``
(trainer.cpp:390), ``Trainer.train_sentences`` ≈ ``train_sentence``
(trainer.cpp:332), and the batcher primitives ``keep_probs`` / ``table`` /
``assemble_batch`` / ``lr_at`` / ``analytic_traffic`` with the reference's
contracts (corpus.cpp:221, sampler.cpp:9-63, model.cpp:39, traffic.cpp:21).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field, fields

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.environ.get("FW2V_LIB") or os.path.join(LIB_DIR, "libfw2v.so")  # FW2V_LIB: experiment builds
DROPIN_PATH = os.path.join(LIB_DIR, "libringvec_fw2v.so")

REUSE_MODES = {"lifetime": 0, "window": 1, "none": 2, "window_snapshot": 3}
SAMPLERS = {"reference": 0, "alias": 1}
MERGES = {"mean": 0, "touched": 1}

OK = 0
ERR_NO_DEVICE = 66
ERR_CUDA = 64
ERR_UNSUPPORTED = 65
ERR_BAD_ARGUMENT = 4
ERR_BAD_CONFIG = 5

# Every symbol include/fw2v.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "fw2v_abi_version", "fw2v_last_error", "fw2v_config_default", "fw2v_validate_config",
    "fw2v_device_count", "fw2v_create", "fw2v_destroy", "fw2v_get_model", "fw2v_set_model",
    "fw2v_init_model", "fw2v_model_device", "fw2v_attach_model", "fw2v_row_stride",
    "fw2v_train_corpus", "fw2v_train_sentences", "fw2v_plan_epoch", "fw2v_plan_info",
    "fw2v_plan_run", "fw2v_plan_destroy", "fw2v_keep_probs", "fw2v_table_build",
    "fw2v_assemble_batch", "fw2v_lr_at", "fw2v_analytic_traffic", "fw2v_corpus_synth_zipf",
    "fw2v_corpus_view", "fw2v_corpus_free", "fw2v_write_embeddings", "fw2v_save_model",
    "fw2v_nearest_neighbors", "fw2v_eval_analogy", "fw2v_alias_draws", "fw2v_plan_chunks",
    "fw2v_average", "fw2v_nccl_unique_id", "fw2v_comm_init_rank", "fw2v_train_corpus_multi",
    "fw2v_merge_begin", "fw2v_merge_replicas", "fw2v_release_cached",
]


class Fw2vError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fw2v error {code}: {msg}")
        self.code = code


class CConfig(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("window", C.c_int32), ("negatives", C.c_int32), ("epochs", C.c_int32),
        ("alpha0", C.c_float), ("subsample", C.c_double),
        ("min_count", C.c_uint64), ("batch_sentences", C.c_uint64), ("max_sentence_len", C.c_uint64),
        ("workers", C.c_int32), ("seed", C.c_uint64), ("reuse_mode", C.c_int32),
        ("table_power", C.c_double), ("table_size", C.c_uint64), ("queue_capacity", C.c_uint64),
        ("ignore_delimiters", C.c_int32),
        ("device", C.c_int32), ("deterministic", C.c_int32), ("sampler", C.c_int32),
        ("fast_sigmoid", C.c_int32), ("k1_lanes", C.c_int32), ("streams", C.c_int32),
        ("l1_refresh_log2", C.c_int32), ("delta_writeback", C.c_int32), ("max_inflight", C.c_int32),
        ("hot_rows", C.c_int32), ("hot_replicas", C.c_int32), ("replica_merge", C.c_int32),
        ("divergence_guard", C.c_int32), ("hot_merge", C.c_int32),
    ]


class CCounters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("context_reads", "context_writes", "sample_reads",
                                          "sample_writes", "ring_hits", "words", "sentences")]

    def as_tuple(self):
        return (self.context_reads, self.context_writes, self.sample_reads, self.sample_writes,
                self.ring_hits)


class CEpoch(C.Structure):
    _fields_ = [("epoch", C.c_int32), ("words", C.c_uint64), ("seconds", C.c_double),
                ("words_per_sec", C.c_double)]


class CReport(C.Structure):
    _fields_ = [
        ("words_trained", C.c_uint64), ("sentences_trained", C.c_uint64), ("vocab_size", C.c_uint64),
        ("wall_seconds", C.c_double), ("batching_words_per_sec", C.c_double), ("n_epochs", C.c_int32),
        ("traffic", CCounters), ("analytic", CCounters), ("kernel_seconds", C.c_double),
        ("h2d_bytes", C.c_uint64), ("guard_retries", C.c_int32),
    ]


OBSERVER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint64)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), C.c_int32, C.c_uint64,
                          C.POINTER(C.c_uint64))
EPOCH_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(CEpoch))


@dataclass
class TrainConfig:
    """ringvec::TrainConfig (config.hpp:13-35) plus the B200 extension."""

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
    # ---- B200 extension ----
    device: int = 0
    deterministic: int = -1
    sampler: str = "reference"
    fast_sigmoid: bool = True
    k1_lanes: int = 0
    streams: int = 0
    l1_refresh_log2: int = 5
    delta_writeback: int = 2  # 2 Hogwild overwrite (K1s: no smem ring), 1 red.add delta, 0 exact overwrite order
    max_inflight: int = 0
    hot_rows: int = 64
    hot_replicas: int = 16
    replica_merge: str = "touched"  # data-parallel rounds: mean | touched (include/fw2v.h)
    divergence_guard: int = 1  # Hogwild: finite check per epoch, restore + halve in-flight on failure
    hot_merge: int = 1  # hot-row replicas: 1 live sum (full Hogwild step), 0 mean at the end of each pass

    @property
    def context_width(self) -> int:
        return (self.window + 1) // 2

    def to_c(self) -> CConfig:
        c = CConfig()
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "reuse_mode":
                v = REUSE_MODES[v]
            elif f.name == "sampler":
                v = SAMPLERS[v]
            elif f.name == "replica_merge":
                v = MERGES[v]
            elif isinstance(v, bool):
                v = int(v)
            setattr(c, f.name, v)
        return c


@dataclass
class Report:
    words_trained: int
    sentences_trained: int
    wall_seconds: float
    batching_words_per_sec: float
    traffic: tuple
    analytic: tuple
    h2d_bytes: int
    epochs: list = field(default_factory=list)
    kernel_seconds: float = 0.0
    guard_retries: int = 0


_lib = None


def _prefer_torch_nccl():
    """libfw2v opens NCCL lazily (dlopen "libnccl.so.2"). In a Python process
    that may import torch, it must be torch's bundled copy: once a library with
    that soname is loaded, torch's own libtorch_cuda binds to it, and the
    system 2.27 lacks symbols torch needs. FW2V_NCCL_LIB points libfw2v at it."""
    if os.environ.get("FW2V_NCCL_LIB"):
        return
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for root in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(root, "nccl", "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["FW2V_NCCL_LIB"] = cand
            return


def lib() -> C.CDLL:
    """Loads libfw2v.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` or __graft_entry__.build()")
    _prefer_torch_nccl()
    L = C.CDLL(LIB_PATH)
    L.fw2v_last_error.restype = C.c_char_p
    L.fw2v_lr_at.restype = C.c_float
    L.fw2v_lr_at.argtypes = [C.c_uint64, C.c_uint64, C.c_float]
    L.fw2v_assemble_batch.restype = C.c_int64
    L.fw2v_row_stride.restype = C.c_int32
    L.fw2v_destroy.restype = None
    L.fw2v_plan_destroy.restype = None
    L.fw2v_corpus_free.restype = None
    _lib = L
    return L


def _check(rc: int):
    if rc != OK:
        raise Fw2vError(rc, lib().fw2v_last_error().decode())


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def device_count() -> int:
    n = C.c_int(0)
    lib().fw2v_device_count(C.byref(n))
    return n.value


def row_stride(cfg: TrainConfig) -> int:
    c = cfg.to_c()
    return lib().fw2v_row_stride(C.byref(c))


# ------------------------------------------------------------ batcher primitives
def keep_probs(counts, threshold):
    counts = np.ascontiguousarray(counts, np.uint64)
    out = np.zeros(len(counts), np.float64)
    on = lib().fw2v_keep_probs(_p(counts, C.c_uint64), len(counts), C.c_double(threshold), _p(out, C.c_double))
    return out if on else None


def table(counts, power, size):
    counts = np.ascontiguousarray(counts, np.uint64)
    out = np.zeros(size, np.int32)
    _check(lib().fw2v_table_build(_p(counts, C.c_uint64), len(counts), C.c_double(power), C.c_uint64(size),
                                  _p(out, C.c_int32)))
    return out


def assemble_batch(counts, offsets, ids, cursor, max_sentences, negatives, power, table_size, threshold,
                   seed, a, b, c):
    counts = np.ascontiguousarray(counts, np.uint64)
    offsets = np.ascontiguousarray(offsets, np.uint64)
    ids = np.ascontiguousarray(ids, np.int32)
    cap = len(ids) + 1
    o_ids = np.zeros(cap, np.int32)
    o_off = np.zeros(len(offsets) + 1, np.uint64)
    o_negs = np.zeros(cap * max(negatives, 1), np.int32)
    cur = C.c_uint64(cursor)
    n = lib().fw2v_assemble_batch(
        _p(counts, C.c_uint64), len(counts), _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1),
        _p(ids, C.c_int32), C.byref(cur), C.c_uint64(max_sentences), negatives, C.c_double(power),
        C.c_uint64(table_size), C.c_double(threshold), C.c_uint64(seed), C.c_uint64(a), C.c_uint64(b),
        C.c_uint64(c), _p(o_ids, C.c_int32), _p(o_off, C.c_uint64), _p(o_negs, C.c_int32))
    if n < 0:
        _check(-n)
    off = o_off[: n + 1].copy()
    w = int(off[-1])
    return cur.value, off, o_ids[:w].copy(), o_negs[: w * negatives].copy()


def alias_draws(counts, power, seed, count):
    counts = np.ascontiguousarray(counts, np.uint64)
    out = np.zeros(max(count, 1), np.int32)
    _check(lib().fw2v_alias_draws(_p(counts, C.c_uint64), len(counts), C.c_double(power), C.c_uint64(seed),
                                  C.c_uint64(count), _p(out, C.c_int32)))
    return out[:count]


def lr_at(trained, total, alpha0):
    return lib().fw2v_lr_at(trained, total, alpha0)


def analytic_traffic(length, width, negatives, mode="lifetime"):
    c = CCounters()
    _check(lib().fw2v_analytic_traffic(C.c_uint64(length), width, negatives, REUSE_MODES[mode], C.byref(c)))
    return c.as_tuple()


# ------------------------------------------------------------ synthetic corpora
def _token_blob(tokens):
    enc = [t.encode() if isinstance(t, str) else bytes(t) for t in tokens]
    offs = np.zeros(len(enc) + 1, np.uint64)
    offs[1:] = np.cumsum([len(e) for e in enc])
    blob = C.create_string_buffer(b"".join(enc), int(offs[-1]) + 1)
    return blob, offs


def write_embeddings(path, rows, tokens, threads=0):
    """save_embeddings (model.cpp:47-74) byte for byte, on all host cores."""
    rows = np.ascontiguousarray(rows, np.float32)
    if rows.ndim != 2 or rows.shape[0] != len(tokens):
        raise ValueError("rows must be |V| x dim with one token per row")
    blob, offs = _token_blob(tokens)
    _check(lib().fw2v_write_embeddings(_p(rows, C.c_float), rows.shape[0], rows.shape[1], C.c_int64(rows.shape[1]),
                                       blob, _p(offs, C.c_uint64), os.fsencode(path), threads))


def nearest_neighbors(rows, queries, k):
    """nearest_neighbors (eval.cpp:303-348) on the GPU for many query ids: (ids, cos), each |Q| x k."""
    rows = np.ascontiguousarray(rows, np.float32)
    q = np.ascontiguousarray(queries, np.int32)
    ids = np.zeros((len(q), k), np.int32)
    cos = np.zeros((len(q), k), np.float64)
    _check(lib().fw2v_nearest_neighbors(_p(rows, C.c_float), rows.shape[0], rows.shape[1], _p(q, C.c_int32), len(q), k,
                                        _p(ids, C.c_int32), _p(cos, C.c_double)))
    return ids, cos


def eval_analogy(rows, quads, method="cos_add"):
    """eval_analogy (eval.cpp:212-290) on the GPU: (predicted ids, accuracy) for |Q| x 4 id quadruples."""
    rows = np.ascontiguousarray(rows, np.float32)
    qd = np.ascontiguousarray(quads, np.int32).reshape(-1, 4)
    pred = np.zeros(len(qd), np.int32)
    _check(lib().fw2v_eval_analogy(_p(rows, C.c_float), rows.shape[0], rows.shape[1], _p(qd, C.c_int32), len(qd),
                                   {"cos_add": 0, "cos_mul": 1}[method], _p(pred, C.c_int32)))
    return pred, float((pred == qd[:, 3]).mean()) if len(qd) else 0.0


class Corpus:
    """Pre-subsampling corpus: vocabulary counts (id order), sentence offsets, ids."""

    def __init__(self, counts, offsets, ids, _handle=None):
        self.counts = counts
        self.offsets = offsets
        self.ids = ids
        self._handle = _handle

    @property
    def n_sentences(self):
        return len(self.offsets) - 1

    def __del__(self):
        if getattr(self, "_handle", None) is not None and _lib is not None:
            _lib.fw2v_corpus_free(self._handle)
            self._handle = None

    def head(self, n_sentences: int) -> "Corpus":
        """First n sentences (a bounded sample for CPU baselines); same vocabulary."""
        off = np.ascontiguousarray(self.offsets[: n_sentences + 1])
        c = Corpus(self.counts, off, self.ids[: int(off[-1])])
        c._parent = self  # the views borrow this corpus's C buffers
        return c


def synth_zipf(types, tokens, s=1.0, sentence_len=1000, min_count=5, threads=0) -> Corpus:
    """Zipf corpus of the BASELINE.md shapes, generated by libfw2v (C++)."""
    h = C.c_void_p()
    _check(lib().fw2v_corpus_synth_zipf(C.c_uint64(types), C.c_uint64(tokens), C.c_double(s),
                                        C.c_uint64(sentence_len), C.c_uint64(min_count), threads, C.byref(h)))
    pc, po, pi = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)(), C.POINTER(C.c_int32)()
    v, ns, ni = C.c_int32(), C.c_uint64(), C.c_uint64()
    lib().fw2v_corpus_view(h, C.byref(pc), C.byref(v), C.byref(po), C.byref(ns), C.byref(pi), C.byref(ni))
    counts = np.ctypeslib.as_array(pc, shape=(v.value,))
    offsets = np.ctypeslib.as_array(po, shape=(ns.value + 1,))
    ids = np.ctypeslib.as_array(pi, shape=(max(ni.value, 1),))[: ni.value]
    return Corpus(counts, offsets, ids, _handle=h)


TEXT8_SHAPE = dict(types=71_291, tokens=16_718_845)
ONEBW_SHAPE = dict(types=555_514, tokens=804_269_957)


# ------------------------------------------------------------ trainer
class Trainer:
    """One B200 trainer context (fw2v_ctx): model in HBM, host batcher, streams."""

    def __init__(self, cfg: TrainConfig, counts):
        self.cfg = cfg
        self.counts = np.ascontiguousarray(counts, np.uint64)
        self.vocab = len(self.counts)
        self._c = cfg.to_c()
        h = C.c_void_p()
        _check(lib().fw2v_create(C.byref(self._c), _p(self.counts, C.c_uint64), self.vocab, C.byref(h)))
        self._h = h
        self.stride = row_stride(cfg)

    def close(self):
        if getattr(self, "_h", None):
            lib().fw2v_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def get_model(self):
        d = self.cfg.dim
        i = np.zeros((self.vocab, d), np.float32)
        o = np.zeros((self.vocab, d), np.float32)
        _check(lib().fw2v_get_model(self._h, _p(i, C.c_float), _p(o, C.c_float)))
        return i, o

    def set_model(self, inp=None, out=None):
        pi = _p(np.ascontiguousarray(inp, np.float32), C.c_float) if inp is not None else None
        po = _p(np.ascontiguousarray(out, np.float32), C.c_float) if out is not None else None
        keep = (inp, out)  # noqa: F841 - keep buffers alive across the call
        _check(lib().fw2v_set_model(self._h, pi, po))

    def init_model(self, seed):
        _check(lib().fw2v_init_model(self._h, C.c_uint64(seed)))

    def save_model(self, path, tokens, which="input", threads=0):
        """save_embeddings (model.cpp:47-74) of the device model; which: input | output."""
        if len(tokens) != self.vocab:
            raise ValueError("one token per vocabulary id")
        blob, offs = _token_blob(tokens)
        _check(lib().fw2v_save_model(self._h, {"input": 0, "output": 1}[which], blob, _p(offs, C.c_uint64),
                                     os.fsencode(path), threads))

    def model_device(self):
        s0, s1, st = C.c_void_p(), C.c_void_p(), C.c_int32()
        _check(lib().fw2v_model_device(self._h, C.byref(s0), C.byref(s1), C.byref(st)))
        return s0.value, s1.value, st.value

    def attach_model(self, syn0_ptr: int, syn1_ptr: int):
        _check(lib().fw2v_attach_model(self._h, C.c_void_p(syn0_ptr), C.c_void_p(syn1_ptr)))

    def train_sentences(self, offsets, ids, negatives, alphas, serial=True):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        ids = np.ascontiguousarray(ids, np.int32)
        negatives = np.ascontiguousarray(negatives, np.int32)
        if negatives.size == 0:
            negatives = np.zeros(1, np.int32)
        alphas = np.ascontiguousarray(alphas, np.float32)
        c = CCounters()
        _check(lib().fw2v_train_sentences(self._h, _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1),
                                          _p(ids, C.c_int32), _p(negatives, C.c_int32),
                                          _p(alphas, C.c_float), int(serial), C.byref(c)))
        return c

    def train_corpus(self, corpus: Corpus, observer=None, on_epoch=None) -> Report:
        offsets = np.ascontiguousarray(corpus.offsets, np.uint64)
        ids = np.ascontiguousarray(corpus.ids, np.int32)
        epochs = []

        def _ep(_u, st):
            e = st.contents
            epochs.append(dict(epoch=e.epoch, words=e.words, seconds=e.seconds, words_per_sec=e.words_per_sec))
            if on_epoch:
                on_epoch(epochs[-1])

        cb_obs = OBSERVER_FN(lambda _u, s, t: observer(s, t)) if observer else OBSERVER_FN()
        cb_ep = EPOCH_FN(_ep)
        rep = CReport()
        _check(lib().fw2v_train_corpus(self._h, _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1),
                                       _p(ids, C.c_int32), cb_obs, None, cb_ep, None, C.byref(rep)))
        return _report(rep, epochs)

    def plan_chunks(self, corpus: Corpus, n_chunks: int, chunk_begin: int, chunk_end: int, epoch: int = 0,
                    words_base: int = 0, words_scale: int = 1) -> "Plan":
        """Device-resident batches of chunks [chunk_begin, chunk_end) of an n_chunks partition
        (one shard / one averaging round of a data-parallel job; fw2v_plan_chunks)."""
        offsets = np.ascontiguousarray(corpus.offsets, np.uint64)
        ids = np.ascontiguousarray(corpus.ids, np.int32)
        h = C.c_void_p()
        _check(lib().fw2v_plan_chunks(self._h, _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1),
                                      _p(ids, C.c_int32), epoch, n_chunks, chunk_begin, chunk_end,
                                      C.c_uint64(words_base), words_scale, C.byref(h)))
        return Plan(self, h)

    def comm_init_rank(self, unique_id: bytes, world: int, rank: int):
        """Joins a cross-process NCCL communicator (fw2v_comm_init_rank)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib().fw2v_comm_init_rank(self._h, buf, world, rank))

    def plan_epoch(self, corpus: Corpus, epoch: int = 0) -> "Plan":
        offsets = np.ascontiguousarray(corpus.offsets, np.uint64)
        ids = np.ascontiguousarray(corpus.ids, np.int32)
        h = C.c_void_p()
        _check(lib().fw2v_plan_epoch(self._h, _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1),
                                     _p(ids, C.c_int32), epoch, C.byref(h)))
        return Plan(self, h)


def _report(rep, epochs) -> Report:
    return Report(rep.words_trained, rep.sentences_trained, rep.wall_seconds, rep.batching_words_per_sec,
                  rep.traffic.as_tuple(), rep.analytic.as_tuple(), rep.h2d_bytes, epochs, rep.kernel_seconds,
                  rep.guard_retries)


def _handles(trainers):
    arr = (C.c_void_p * len(trainers))(*[t._h for t in trainers])
    return arr


def average(trainers):
    """Replica average over trainers (fw2v_average): NCCL across devices, peer kernel otherwise."""
    _check(lib().fw2v_average(_handles(trainers), len(trainers)))


def _exchange_cb(exchange):
    def _ex(_u, bufs, counts, n_bufs, local, out):
        try:
            out[0] = int(exchange([(bufs[i], counts[i]) for i in range(n_bufs)], int(local)))
            return 0
        except Exception:  # noqa: BLE001 - reported through the status code
            import traceback

            traceback.print_exc()
            return ERR_BAD_ARGUMENT

    return EXCHANGE_FN(_ex) if exchange else EXCHANGE_FN()


def merge_begin(trainers):
    _check(lib().fw2v_merge_begin(_handles(trainers), len(trainers)))


def merge_replicas(trainers, local_words, n_shards=0, exchange=None) -> int:
    """One replica merge (fw2v_merge_replicas); returns the global word count."""
    lw = np.ascontiguousarray(local_words, np.uint64)
    g = C.c_uint64()
    cb = _exchange_cb(exchange)
    _check(lib().fw2v_merge_replicas(_handles(trainers), len(trainers), n_shards or len(trainers), _p(lw, C.c_uint64),
                                     cb, None, C.byref(g)))
    return g.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().fw2v_nccl_unique_id(buf))
    return bytes(buf)


def train_corpus_multi(trainers, corpus: Corpus, average_words: int = 0, shard0: int = 0, n_shards: int = 0,
                       exchange=None, on_epoch=None) -> Report:
    """Data-parallel training (fw2v_train_corpus_multi): trainer i trains shard shard0+i of n_shards
    (default: len(trainers)). exchange(buffers, local_words) -> global_words connects processes:
    `buffers` are (device pointer, float count) pairs it must SUM over the processes in place."""
    offsets = np.ascontiguousarray(corpus.offsets, np.uint64)
    ids = np.ascontiguousarray(corpus.ids, np.int32)
    epochs = []

    def _ep(_u, st):
        e = st.contents
        epochs.append(dict(epoch=e.epoch, words=e.words, seconds=e.seconds, words_per_sec=e.words_per_sec))
        if on_epoch:
            on_epoch(epochs[-1])

    cb_ep = EPOCH_FN(_ep)
    cb_ex = _exchange_cb(exchange)
    rep = CReport()
    _check(lib().fw2v_train_corpus_multi(_handles(trainers), len(trainers), shard0, n_shards or len(trainers),
                                         _p(offsets, C.c_uint64), C.c_uint64(len(offsets) - 1), _p(ids, C.c_int32),
                                         C.c_uint64(average_words), cb_ex, None, OBSERVER_FN(), None, cb_ep, None,
                                         C.byref(rep)))
    return _report(rep, epochs)


class CHarnessConfig(C.Structure):
    _fields_ = CConfig._fields_[:16]


class CHarnessResult(C.Structure):
    _fields_ = [("call_seconds", C.c_double), ("epoch_words_per_sec", C.c_double), ("words_trained", C.c_uint64),
                ("input_checksum", C.c_double)]


HARNESS_PATH = os.path.join(LIB_DIR, "libringvec_harness.so")


class DropinHarness:
    """A reference-side caller of the ringvec::train drop-in (libringvec_harness.so,
    csrc/ringvec_harness.cpp): holds a ringvec::Corpus and times whole train() calls."""

    def __init__(self, corpus: Corpus):
        if not os.path.exists(HARNESS_PATH):
            raise ImportError(f"{HARNESS_PATH} missing: `make harness` (needs the reference sources)")
        lib()  # FW2V_NCCL_LIB before the drop-in can open NCCL
        self.L = C.CDLL(HARNESS_PATH)
        self.L.fw2v_harness_last_error.restype = C.c_char_p
        self.L.fw2v_harness_free.restype = None
        offsets = np.ascontiguousarray(corpus.offsets, np.uint64)
        ids = np.ascontiguousarray(corpus.ids, np.int32)
        counts = np.ascontiguousarray(corpus.counts, np.uint64)
        h = C.c_void_p()
        self._check(self.L.fw2v_harness_corpus(_p(counts, C.c_uint64), len(counts), _p(offsets, C.c_uint64),
                                               C.c_uint64(len(offsets) - 1), _p(ids, C.c_int32), C.byref(h)))
        self.h = h

    def _check(self, rc):
        if rc != 0:
            raise Fw2vError(rc, self.L.fw2v_harness_last_error().decode())

    def train(self, cfg: TrainConfig):
        """One ringvec::train(corpus, cfg) call (reference TrainConfig fields of cfg; GPU
        knobs come from FW2V_* environment variables as for any drop-in user)."""
        full = cfg.to_c()
        hc = CHarnessConfig()
        for name, _ in CHarnessConfig._fields_:
            setattr(hc, name, getattr(full, name))
        r = CHarnessResult()
        self._check(self.L.fw2v_harness_train(self.h, C.byref(hc), C.byref(r)))
        return r

    def close(self):
        if getattr(self, "h", None):
            self.L.fw2v_harness_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Plan:
    """One epoch of batches resident in HBM (fw2v_plan)."""

    def __init__(self, trainer: Trainer, handle):
        self.trainer = trainer
        self._h = handle
        w, s, b, by = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib().fw2v_plan_info(handle, C.byref(w), C.byref(s), C.byref(b), C.byref(by))
        self.words, self.sentences, self.batches, self.device_bytes = w.value, s.value, b.value, by.value

    def run(self):
        """Launches the plan's kernels; returns (device seconds, counters)."""
        sec = C.c_double()
        c = CCounters()
        _check(lib().fw2v_plan_run(self.trainer._h, self._h, C.byref(sec), C.byref(c)))
        return sec.value, c

    def close(self):
        if getattr(self, "_h", None):
            lib().fw2v_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
