#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_hot_live.py tests/test_multi_gpu.py tests/test_guard.py tests/test_observer.py tests/test_reference_suite.py -q -x -s 2>&1 | grep -E "passed|failed|Error|dp2|gloo|assert" | tail -20
timeout 600 python tools/dropin_probe.py 2>&1 | head -8
