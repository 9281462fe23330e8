#!/bin/bash
# ncu launch lists of one bench step per update order (and the 1bw shape), then
# profiles/bench_roofline.json for bench.py's roofline block.
# usage: tools/bench_profiles.sh TAG
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${1:-r02}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,smsp__inst_executed.sum
./tools/l2_bw > gpurun_out/l2bw_$TAG.txt 2>&1
ARGS=""
for spec in "window_snapshot text8" "lifetime text8" "window_snapshot 1bw" "lifetime 1bw"; do
  set -- $spec
  timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
     --log-file gpurun_out/step_$1_$2_$TAG.csv python tools/ncu_bench_step.py $1 $2 > gpurun_out/step_$1_$2_$TAG.log 2>&1
  W=$(grep -o "words [0-9]*" gpurun_out/step_$1_$2_$TAG.log | awk '{print $2}')
  [ "$2" = "text8" ] && ARGS="$ARGS $1=gpurun_out/step_$1_$2_$TAG.csv:$W"
  [ "$2" = "1bw" ] && ARGS="$ARGS $1_1bw=gpurun_out/step_$1_$2_$TAG.csv:$W"
done
python tools/ncu_bench_summary.py gpurun_out/bench_roofline_$TAG.json gpurun_out/l2bw_$TAG.txt $ARGS
