#!/bin/bash
# Bench line + ncu evidence for one K1s update order (one GPU); summaries are
# made on the box so only text comes back (plus one .ncu-rep < 64 MiB).
# usage: tools/final_profiles.sh TAG MODE [bench]
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${1:-r01j}; MODE=${2:-window_snapshot}
mkdir -p gpurun_out
if [ "$3" = "bench" ]; then
  timeout 400 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
  tail -1 gpurun_out/bench_$TAG.json | cut -c1-200
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
fi
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1s -s 1 -c 1 -o gpurun_out/full_${MODE}_$TAG -f \
  python tools/ncu_probe.py $MODE 20000 128 1 > gpurun_out/ncu_${MODE}_$TAG.log 2>&1
python tools/ncu_quick.py gpurun_out/full_${MODE}_$TAG.ncu-rep 9897591 > gpurun_out/quick_${MODE}_$TAG.txt 2>&1
python tools/ncu_lines.py gpurun_out/full_${MODE}_$TAG.ncu-rep 9897591 60 > gpurun_out/lines_${MODE}_$TAG.txt 2>&1
head -12 gpurun_out/quick_${MODE}_$TAG.txt
du -sh gpurun_out
