#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stair.py -x -q -k hogwild -s 2>&1 | grep -E "hot_rows|passed|failed" > gpurun_out/pytest_r02e.log; cat gpurun_out/pytest_r02e.log
bash tools/final_profiles.sh r02e lifetime
bash tools/final_profiles.sh r02e window_snapshot
