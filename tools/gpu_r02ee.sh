#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash tools/bench_profiles.sh r02ee > gpurun_out/bench_profiles_r02ee.log 2>&1; tail -3 gpurun_out/bench_profiles_r02ee.log
bash tools/final_profiles.sh r02ee window_snapshot > /dev/null 2>&1; head -12 gpurun_out/quick_window_snapshot_r02ee.txt
bash tools/gpu_l2split.sh > gpurun_out/l2split_r02ee.txt 2>&1; grep -E "==|srcunit_tex.sum|op_red.sum|gpu__time" gpurun_out/l2split_r02ee.txt
rm -f gpurun_out/*.ncu-rep
