"""Data-parallel replicas on the B200 box's one GPU.

The product path is native (fw2v_train_corpus_multi + fw2v_average, include/
fw2v.h). Every gpurun box has one GPU, so the replicas here share device 0:
fw2v_average then takes its peer-memory kernel path (NCCL refuses two ranks on
one device), and the cross-process leg runs two processes with a gloo exchange
callback. The NCCL path itself is exercised with a one-rank communicator.
"""
import os
import socket

import numpy as np
import pytest

from helpers import sgns_loss

pytestmark = pytest.mark.gpu
fw = pytest.importorskip("paper_2312_07743_b200")
from oracle.oracle import TrainConfig as RConfig  # noqa: E402

from paper_2312_07743_b200.dist import dp_chunks  # noqa: E402


def test_average_peer_kernel_is_the_mean():
    V, d = 1000, 128
    counts = (5000 - np.arange(V)).astype(np.uint64)
    ts = [fw.Trainer(fw.TrainConfig(dim=d, seed=s, workers=4, deterministic=0), counts) for s in (1, 2, 3)]
    try:
        ms = [t.get_model() for t in ts]
        rng = np.random.default_rng(0)
        for t in ts:  # non-zero output matrices too
            t.set_model(None, rng.standard_normal((V, d)).astype(np.float32))
        outs = [t.get_model()[1] for t in ts]
        fw.average(ts)
        want_in = ((ms[0][0] + ms[1][0]) + ms[2][0]) * np.float32(1.0 / 3.0)
        want_out = ((outs[0] + outs[1]) + outs[2]) * np.float32(1.0 / 3.0)
        for t in ts:
            gi, go = t.get_model()
            np.testing.assert_array_equal(gi, want_in)
            np.testing.assert_array_equal(go, want_out)
        fw.average(ts[:1])  # one replica: no-op
        np.testing.assert_array_equal(ts[0].get_model()[0], want_in)
    finally:
        for t in ts:
            t.close()


def test_average_rejects_mismatched_replicas():
    a = fw.Trainer(fw.TrainConfig(dim=32, workers=4, deterministic=0), np.arange(100, 0, -1).astype(np.uint64))
    b = fw.Trainer(fw.TrainConfig(dim=64, workers=4, deterministic=0), np.arange(100, 0, -1).astype(np.uint64))
    with a, b:
        with pytest.raises(fw.Fw2vError) as e:
            fw.average([a, b])
        assert e.value.code == fw.fw2v.ERR_BAD_ARGUMENT


def test_nccl_one_rank_communicator():
    """The NCCL path (dlopen'd libnccl, ncclCommInitRank, ncclAllReduce/ncclAvg)
    with a one-rank communicator: the average is the identity."""
    counts = (3000 - np.arange(500)).astype(np.uint64)
    with fw.Trainer(fw.TrainConfig(dim=64, workers=4, deterministic=0), counts) as t:
        before = t.get_model()
        t.comm_init_rank(fw.nccl_unique_id(), 1, 0)
        fw.average([t])
        after = t.get_model()
    np.testing.assert_array_equal(before[0], after[0])
    np.testing.assert_array_equal(before[1], after[1])


TEXT8_CFG = dict(dim=128, window=5, negatives=5, epochs=1, batch_sentences=10000, subsample=1e-4, seed=1)


def _text8_loss_fn(c):
    p = c.counts.astype(np.float64) ** 0.75
    negs = np.random.default_rng(5).choice(len(c.counts), 400_000 * 5, p=p / p.sum()).astype(np.int32)
    off = c.offsets[:401].copy()

    def loss(inp, out):
        return sgns_loss(inp, out, off, c.ids[: int(off[-1])], negs, wf=3, n_neg=5, max_pairs=100_000)

    return loss


@pytest.fixture(scope="module")
def text8_ref(ref):
    """The reference trainer with 16 producers on the text8 shape, one epoch."""
    c = fw.synth_zipf(**fw.TEXT8_SHAPE)
    inp, out, rep = ref.train(c.counts, c.offsets, c.ids, RConfig(workers=16, **TEXT8_CFG))
    loss = _text8_loss_fn(c)
    return c, loss, loss(inp, out), rep


@pytest.mark.parametrize("mode", ["lifetime", "window_snapshot"])
@pytest.mark.parametrize("sampler", ["reference", "alias"])
@pytest.mark.parametrize("merge", ["touched", "mean"])
def test_train_multi_two_replicas(text8_ref, mode, sampler, merge):
    """Two replicas, each a contiguous shard, merged twice per epoch: the union
    of their batches is the reference's for workers=16 (exact global word and
    sentence counts), and the SGNS loss matches the reference within the tier-2
    tolerance. (Data-parallel quality needs words per replica: on the 3 M-token
    planted corpus 2 replicas already cost +4.4%, profiles/r02_dp_merge_probe.txt.)"""
    c, loss_fn, ref_loss, rrep = text8_ref
    est = rrep.words_trained / 2  # words per shard and epoch
    cfg = fw.TrainConfig(workers=16, deterministic=0, reuse_mode=mode, sampler=sampler, replica_merge=merge,
                         **TEXT8_CFG)
    ts = [fw.Trainer(cfg, c.counts) for _ in range(2)]
    try:
        rep = fw.train_corpus_multi(ts, c, average_words=int(est / 2))
        m = [t.get_model() for t in ts]
    finally:
        for t in ts:
            t.close()
    assert dp_chunks(16, 2, 2)[0] == 16  # same partition as the reference's 16 producers
    assert rep.words_trained == rrep.words_trained
    assert rep.sentences_trained == rrep.sentences_trained
    assert rep.traffic == rep.analytic
    np.testing.assert_array_equal(m[0][0], m[1][0])  # replicas equal after the final merge
    np.testing.assert_array_equal(m[0][1], m[1][1])
    loss = loss_fn(m[0][0], m[0][1])
    print(f"dp2 {mode} {sampler} {merge}: loss {loss:.4f} vs ref {ref_loss:.4f}")
    assert abs(loss - ref_loss) / ref_loss <= 0.02


def test_train_multi_rejects_deterministic():
    counts = (3000 - np.arange(50)).astype(np.uint64)
    with fw.Trainer(fw.TrainConfig(dim=16, workers=1), counts) as a, fw.Trainer(fw.TrainConfig(dim=16, workers=1),
                                                                                counts) as b:
        c = fw.Corpus(counts, np.array([0, 3], np.uint64), np.array([1, 2, 3], np.int32))
        with pytest.raises(fw.Fw2vError) as e:
            fw.train_corpus_multi([a, b], c)
        assert e.value.code == fw.fw2v.ERR_UNSUPPORTED


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    """One process of a 2-rank job on the box's single GPU: gloo process group,
    native trainer per rank with its model in torch tensors, exchange callback
    averaging them (NCCL cannot put two ranks on one device)."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2312_07743_b200 as fw_
    from paper_2312_07743_b200.dist import TorchExchange
    from test_multi_gpu import TEXT8_CFG

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = fw_.synth_zipf(**fw_.TEXT8_SHAPE)
        cfg = fw_.TrainConfig(workers=16, deterministic=0, reuse_mode="window_snapshot", **TEXT8_CFG)
        t = fw_.Trainer(cfg, c.counts)
        ex = TorchExchange()
        rep = fw_.train_corpus_multi([t], c, average_words=1_200_000, shard0=rank, n_shards=world, exchange=ex)
        gi, go = t.get_model()
        q.put((rank, rep.words_trained, rep.sentences_trained, ex.calls, gi, go))
        t.close()
    finally:
        dist.destroy_process_group()


def test_two_process_gloo_exchange(text8_ref):
    """world_size 2 (two processes, one GPU, gloo): shards, per-round exchange
    (touched merge), global schedule; the job's words equal the reference's and
    its loss is within 2%."""
    import torch.multiprocessing as mp

    c, loss_fn, ref_loss, rrep = text8_ref
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert sum(r[1] for r in res) == rrep.words_trained
    assert sum(r[2] for r in res) == rrep.sentences_trained
    assert res[0][3] >= 4  # merged ~4 times in the epoch
    np.testing.assert_array_equal(res[0][4], res[1][4])
    loss = loss_fn(res[0][4], res[0][5])
    print(f"2-process gloo: loss {loss:.4f} vs ref {ref_loss:.4f}")
    assert abs(loss - ref_loss) / ref_loss <= 0.02
