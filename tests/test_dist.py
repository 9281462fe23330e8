"""Multi-process host logic on CPU (gloo, world_size 2): corpus sharding, the
data-parallel chunk partition, the replica average, the global word count
behind the lr schedule, and the exchange callback the native trainer calls."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_07743_b200.dist import ReplicaAverager, TorchExchange, dp_chunks, global_words, shard_bounds


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


def test_dp_chunks_whole_rounds():
    # workers already a multiple of shards x rounds: the reference's own partition
    assert dp_chunks(16, 2, 2) == (16, 8, 4)
    assert dp_chunks(64, 8, 1) == (64, 8, 8)
    # rounded up so every shard and round holds whole chunks
    assert dp_chunks(10, 4, 1) == (12, 3, 3)
    assert dp_chunks(1, 8, 3) == (24, 3, 1)
    for w in range(1, 40):
        for s in (1, 2, 3, 8):
            for r in (1, 2, 5):
                tot, per_shard, per_round = dp_chunks(w, s, r)
                assert tot >= max(w, s) and tot % (s * r) == 0 and per_shard * s == tot and per_round * r == per_shard
    with pytest.raises(ValueError):
        dp_chunks(0, 1, 1)


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
        # the exchange callback: summands differ per element, words per rank
        rng = np.random.default_rng(rank)
        m2 = torch.from_numpy(rng.standard_normal((2, 7, 12)).astype(np.float32))
        ex = TorchExchange()
        g = ex([m2[0], m2[1]], 123 + rank)
        q.put((rank, model.mean().item(), float(model.std()), words, avg.rounds, m2.numpy().copy(), g, ex.calls))
    finally:
        dist.destroy_process_group()


def test_replica_average_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    want = sum(np.random.default_rng(r).standard_normal((2, 7, 12)).astype(np.float32) for r in range(world))
    for rank, mean, std, words, rounds, m2, g, calls in res:
        assert mean == pytest.approx(0.5) and std == 0.0
        assert words == 3000 and rounds == 1
        np.testing.assert_allclose(m2, want, rtol=0, atol=1e-6)
        assert g == 123 + 124 and calls == 1
    np.testing.assert_array_equal(res[0][5], res[1][5])  # replicas identical after the exchange
