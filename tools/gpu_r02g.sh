#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash tools/bench_profiles.sh r02g > gpurun_out/bench_profiles_r02g.log 2>&1
tail -40 gpurun_out/bench_profiles_r02g.log
cat gpurun_out/l2bw_r02g.txt
