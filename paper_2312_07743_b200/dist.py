"""Multi-GPU plumbing for the FULL-W2V trainer: one process per GPU.

The path shards naturally: sentences are independent Hogwild
units, so each rank trains its own replica of syn0/syn1neg on a contiguous
sentence range (the reference's producer chunking, trainer.cpp:431-434) and
the only exchange is a periodic replica average — one in-place NCCL
all-reduce with ReduceOp.AVG over both matrices, held in one flat tensor so a
single collective covers the whole model (NVLS on NVSwitch systems).
The learning-rate schedule counts the GLOBAL trained words (all ranks).
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_bounds(n_sentences: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous sentence range of `rank`: chunk = ceil(n / world) (trainer.cpp:431-434)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    chunk = (n_sentences + world - 1) // world
    begin = min(n_sentences, rank * chunk)
    return begin, min(n_sentences, begin + chunk)


@dataclass
class AveragePolicy:
    """Average the replicas every `period_words` words trained per rank."""

    period_words: int

    def due(self, words_since_last: int) -> bool:
        return words_since_last >= self.period_words


class ReplicaAverager:
    """In-place replica averaging of a flat model tensor over a process group.

    `model` holds syn0 and syn1neg back to back (2 x |V| x stride fp32); on the
    NCCL backend this is one ncclAllReduce(ncclAvg) over NVLink. Works on any
    torch.distributed backend (gloo on CPU for tests).
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
