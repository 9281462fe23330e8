#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash tools/bench_profiles.sh r02u > gpurun_out/bench_profiles_r02u.log 2>&1; tail -5 gpurun_out/bench_profiles_r02u.log
bash tools/final_profiles.sh r02u lifetime > /dev/null 2>&1
bash tools/final_profiles.sh r02u window_snapshot > /dev/null 2>&1
head -12 gpurun_out/quick_lifetime_r02u.txt; head -12 gpurun_out/quick_window_snapshot_r02u.txt
bash tools/gpu_l2split.sh > gpurun_out/l2split_r02u.txt 2>&1; cat gpurun_out/l2split_r02u.txt
rm -f gpurun_out/*.ncu-rep
