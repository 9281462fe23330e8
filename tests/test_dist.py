"""Multi-process host logic on CPU (gloo, world_size 2): corpus sharding, the
replica average, and the global word count behind the lr schedule."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_07743_b200.dist import AveragePolicy, ReplicaAverager, global_words, shard_bounds


def test_shard_bounds_cover_and_match_reference_chunking():
    for n in [0, 1, 7, 16719, 804270]:
        for world in [1, 2, 3, 8]:
            spans = [shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            chunk = (n + world - 1) // world  # trainer.cpp:431-434
            assert all(b - a <= chunk for a, b in spans)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_average_policy():
    p = AveragePolicy(period_words=1000)
    assert not p.due(999) and p.due(1000)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # replica r holds value r everywhere; the average is (world-1)/2
        model = torch.full((2, 5, 8), float(rank))
        avg = ReplicaAverager(model)
        avg.average()
        words = global_words(1000 * (rank + 1))
        q.put((rank, model.mean().item(), float(model.std()), words, avg.rounds))
    finally:
        dist.destroy_process_group()


def test_replica_average_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for rank, mean, std, words, rounds in res:
        assert mean == pytest.approx(0.5) and std == 0.0
        assert words == 3000 and rounds == 1
    np.testing.assert_equal(len(res), world)
