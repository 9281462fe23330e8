#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hot_live.py tests/test_gpu_parity.py -q -x -k "live or hot_replicas" 2>&1 | tail -1
for m in window_snapshot lifetime; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode $m 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(j['value']/1e6,1), 'Mw/s')"
done
t0=$(date +%s); timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo "smoke under ncu rc=$? wall $(( $(date +%s) - t0 )) s"; tail -1 gpurun_out/smoke_ncu.log
t0=$(date +%s); timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dropin > gpurun_out/bench_ncu.log 2>&1; echo "bench under ncu rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 1200 python -m pytest tests/test_quality.py -q -s -k "text8_multi or hot_band" 2>&1 | grep -E "text8|passed|failed"
