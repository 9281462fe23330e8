#!/bin/bash
# One GPU call: gpu tests, bench, ncu launch list + full capture of the top kernel.
# usage: tools/gpu_round.sh TAG [skip_tests]
cd $GRAFT_REPO_ROOT
TAG=${1:-rX}
mkdir -p gpurun_out
if [ "$2" != "skip_tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_$TAG.log
  tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 400 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1s -s 1 -c 1 -o gpurun_out/full_$TAG -f \
  python tools/ncu_probe.py window_snapshot 20000 128 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
ls -la gpurun_out
if [ -n "$EXTRA" ]; then
  for a in $EXTRA; do
    timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 ${a//,/ } 2>&1 | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a', round(j['value']/1e6,1), 'Mw/s')"
  done
fi
