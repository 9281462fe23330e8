"""Multi-GPU plumbing for the FULL-W2V trainer: one process per GPU.

The path shards naturally: sentences are independent Hogwild
units, so each GPU trains its own replica of syn0/syn1neg on a contiguous shard
of the corpus (whole chunks of the reference's producer partition,
trainer.cpp:431-434) and the only exchange is a periodic replica average. The
product path for that is native: ``fw2v_train_corpus_multi`` (include/fw2v.h)
runs the rounds, keeps the learning-rate schedule on the GLOBAL word count
(trainer.cpp:479-487) and averages with NCCL (``ncclAllReduce`` / ``ncclAvg``,
in-process over ``ncclCommInitAll`` or across processes after
``fw2v_comm_init_rank``).

This module holds the Python side of a multi-process job: sharding arithmetic
and ``TorchExchange``, the exchange callback for process groups NCCL cannot
serve (gloo on CPU, or several ranks sharing one GPU in tests): it SUMs the
buffers the native trainer hands over with ``torch.distributed`` and sums the
word counts.
"""
from __future__ import annotations


def shard_bounds(n_sentences: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous sentence range of `rank`: chunk = ceil(n / world) (trainer.cpp:431-434)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    chunk = (n_sentences + world - 1) // world
    begin = min(n_sentences, rank * chunk)
    return begin, min(n_sentences, begin + chunk)


def dp_chunks(workers: int, n_shards: int, rounds: int) -> tuple[int, int, int]:
    """The data-parallel chunk partition fw2v_train_corpus_multi uses: the
    reference's `workers` chunks rounded up to a multiple of n_shards x rounds.
    Returns (total chunks, chunks per shard, chunks per round)."""
    if workers < 1 or n_shards < 1 or rounds < 1:
        raise ValueError("workers, n_shards and rounds must be >= 1")
    unit = n_shards * rounds
    total = ((max(workers, n_shards) + unit - 1) // unit) * unit
    return total, total // n_shards, total // n_shards // rounds


class ReplicaAverager:
    """In-place replica averaging of a flat model tensor over a process group.

    `model` holds syn0 and syn1neg back to back (2 x |V| x stride fp32). On the
    NCCL backend this is one all-reduce (AVG); gloo sums and divides.
    """

    def __init__(self, model, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.model = model
        self.group = group
        self.rounds = 0

    def average(self):
        dist = self.dist
        if dist.get_backend(self.group) == "gloo" or not hasattr(dist.ReduceOp, "AVG"):
            if self.model.is_cuda and dist.get_backend(self.group) == "gloo":
                host = self.model.cpu()
                dist.all_reduce(host, op=dist.ReduceOp.SUM, group=self.group)
                self.model.copy_(host.div_(dist.get_world_size(self.group)))
            else:
                dist.all_reduce(self.model, op=dist.ReduceOp.SUM, group=self.group)
                self.model.div_(dist.get_world_size(self.group))
        else:
            dist.all_reduce(self.model, op=dist.ReduceOp.AVG, group=self.group)
        self.rounds += 1


def global_words(local_words: int, group=None) -> int:
    """Sum of trained words over ranks (the global lr_at schedule position)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([local_words], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


class _DeviceView:
    """Zero-copy torch view of a library-owned fp32 device buffer."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def device_tensor(ptr: int, count: int):
    import torch

    return torch.as_tensor(_DeviceView(ptr, count), device="cuda")


class TorchExchange:
    """Exchange callback for ``train_corpus_multi(..., exchange=...)``: SUMs the
    buffers the native trainer hands over (its replicas turned into summands,
    per ``replica_merge``) over the process group in place, and returns the
    global word count. Called after this process's kernels finished. gloo
    reduces through host copies."""

    def __init__(self, group=None):
        self.group = group
        self.calls = 0

    def __call__(self, buffers, local_words: int) -> int:
        import torch
        import torch.distributed as dist

        cuda = torch.cuda.is_available()
        if cuda:
            torch.cuda.synchronize()
        gloo = dist.get_backend(self.group) == "gloo"
        for b in buffers:
            t = b if isinstance(b, torch.Tensor) else device_tensor(*b)
            if gloo and t.is_cuda:
                host = t.cpu()
                dist.all_reduce(host, op=dist.ReduceOp.SUM, group=self.group)
                t.copy_(host)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        if cuda:
            torch.cuda.synchronize()
        self.calls += 1
        return global_words(local_words, self.group)
