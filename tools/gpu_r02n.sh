#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sanitizers.py tests/test_stair.py tests/test_guard.py tests/test_observer.py tests/test_reference_suite.py -q -x -s 2>&1 | grep -E "passed|failed|guard retries|loss stair|Error|error" | tail -15
bash tools/gpu_r02m.sh
