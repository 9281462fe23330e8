#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash tools/bench_profiles.sh r02ff > gpurun_out/bench_profiles_r02ff.log 2>&1; tail -3 gpurun_out/bench_profiles_r02ff.log
