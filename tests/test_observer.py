"""TrainObserver (trainer.hpp:82-87) on the device path: every kernel logs
(sentence, target) before each window it starts — empty windows included, as the
reference calls on_target before every window (trainer.cpp:246) — and the host
replays the log into the observer in the device's processing order. The
reference's own check (test_trainer.cpp:450-471: per sentence the targets arrive
0, 1, 2, ... and their total is words_trained) must hold for every engine."""
import threading

import numpy as np
import pytest

from helpers import random_corpus

pytestmark = pytest.mark.gpu
fw = pytest.importorskip("paper_2312_07743_b200")


@pytest.mark.parametrize("engine", [
    dict(workers=1),  # K2, serial exact
    dict(workers=8, deterministic=0, reuse_mode="lifetime"),  # staircase K1s
    dict(workers=8, deterministic=0, reuse_mode="lifetime", window=9),  # one-window wavefront (W_f = 5)
    dict(workers=8, deterministic=0, reuse_mode="window_snapshot"),  # K1s
    dict(workers=8, deterministic=0, reuse_mode="window"),  # K2 per sentence
    dict(workers=8, deterministic=0, reuse_mode="lifetime", max_inflight=40),  # capped grid-stride launches
], ids=["k2", "stair", "wavefront", "snapshot", "window", "capped"])
def test_observer_order_per_sentence(engine):
    counts, offsets, ids = random_corpus(300, 40, 200, seed=9)
    kw = dict(dim=64, window=5, negatives=5, epochs=2, batch_sentences=64, table_size=10007, subsample=1e-3, seed=4)
    kw.update(engine)
    log = {}
    lock = threading.Lock()
    order = []

    def obs(serial, target):
        with lock:
            log.setdefault(serial, []).append(target)
            order.append((serial, target))

    with fw.Trainer(fw.TrainConfig(**kw), counts) as t:
        rep = t.train_corpus(fw.Corpus(counts, offsets, ids), observer=obs)
    assert log, "observer never called"
    for serial, targets in log.items():
        assert targets == list(range(len(targets))), serial
    assert sum(len(v) for v in log.values()) == rep.words_trained
    assert len(log) == rep.sentences_trained
    if engine.get("workers") == 1:  # serial engine: whole sentences in order
        assert order == sorted(order)
