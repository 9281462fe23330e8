#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_guard.py tests/test_multi_gpu.py tests/test_hot_live.py tests/test_embeddings_io.py -q -x 2>&1 | tail -1
timeout 600 python tools/dropin_phases.py 2>&1 | tail -8
