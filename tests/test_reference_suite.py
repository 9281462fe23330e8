"""The reference's own test suites, compiled from /root/reference by
oracle/Makefile and linked against the B200 drop-in ringvec::train
(paper_2312_07743_b200/_lib/libringvec_fw2v.so): every `train()` call in
test_trainer.cpp and acceptance.cpp runs on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def _run(exe, *args):
    path = os.path.join(REF, exe)
    if not os.path.exists(path):
        pytest.skip(f"{exe} not built (make suite)")
    r = subprocess.run([path, *args], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    return r


def test_reference_trainer_suite_on_b200():
    r = _run("test_trainer_gpu")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "failed: 0" in r.stdout


def test_reference_acceptance_on_b200():
    r = _run("acceptance_gpu")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "[FAIL]" not in r.stdout
