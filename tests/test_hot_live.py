"""Live hot-row merge (fw2v_config.hot_merge = 1, csrc/fw2v_kernels.cu k_hot_live):
the top-K output rows are trained as R replicas (sentence s -> replica s mod R) and a
resident merge block keeps summing every replica's updates into the others during
the pass, so each hot row receives every update — plain Hogwild's step. The
pass-end mean (hot_merge = 0, round 1) gives each update 1/R weight instead.

Exact check on sentences that share no rows (no Hogwild interaction): with the
live merge the model equals the no-replica run up to the merge's float rounding;
with the mean the hot rows' updates are divided by R."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
fw = pytest.importorskip("paper_2312_07743_b200")


def _disjoint_hot_batch(rng, n_sent, hot_k, band, V, n_neg, L):
    """Sentence s uses hot ids {2s, 2s+1} and its own band of cold ids, for its
    tokens and its negatives alike."""
    ids, negs, offs = [], [], [0]
    for s in range(n_sent):
        pool = np.concatenate([[2 * s, 2 * s + 1], hot_k + s * band + np.arange(band)])
        ids.append(rng.choice(pool, L))
        negs.append(rng.choice(pool, L * n_neg))
        offs.append(offs[-1] + L)
    return (np.array(offs, np.uint64), np.concatenate(ids).astype(np.int32),
            np.concatenate(negs).astype(np.int32), np.full(n_sent, 0.025, np.float32))


@pytest.mark.parametrize("mode", ["window_snapshot", "lifetime"])
def test_live_merge_keeps_every_update(mode):
    n_sent, hot_k, band, n_neg, L, d = 32, 64, 40, 5, 60, 128
    V = hot_k + n_sent * band
    counts = (10 + V - np.arange(V)).astype(np.uint64)
    rng = np.random.default_rng(11)
    batch = _disjoint_hot_batch(rng, n_sent, hot_k, band, V, n_neg, L)
    inp = ((rng.random((V, d)) - 0.5) / d).astype(np.float32)
    out = ((rng.random((V, d)) - 0.5) * 0.5).astype(np.float32)
    res = {}
    for name, kw in (("plain", dict(hot_rows=0)), ("live", dict(hot_rows=hot_k, hot_merge=1)),
                     ("mean", dict(hot_rows=hot_k, hot_merge=0))):
        cfg = fw.TrainConfig(dim=d, window=5, negatives=n_neg, workers=4, deterministic=0, reuse_mode=mode,
                             l1_refresh_log2=0, max_inflight=-1, **kw)
        with fw.Trainer(cfg, counts) as t:
            t.set_model(inp, out)
            t.train_sentences(*batch, serial=False)
            res[name] = t.get_model()
    pi, po = res["plain"]
    li, lo = res["live"]
    mi, mo = res["mean"]
    upd = np.abs(po[:hot_k] - out[:hot_k]).max()
    assert upd > 1e-3, "hot rows not trained"
    # live: every update kept (float rounding of the merge only)
    assert np.abs(lo - po).max() <= 1e-5 * max(1.0, np.abs(po).max()), np.abs(lo - po).max()
    assert np.abs(li - pi).max() <= 1e-5, np.abs(li - pi).max()
    # mean: the hot rows' updates are scaled by 1/R (16)
    got = np.abs(mo[:hot_k] - out[:hot_k]).max()
    assert got < 0.2 * upd, (got, upd)
