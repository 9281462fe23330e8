#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_quality.py -q -s -k "other_shapes or d512 or text8" 2>&1 | grep -E "zipf|d300|d512|text8|passed|failed"
timeout 900 python bench.py --no-cpu-baseline --no-dropin --no-e2e --no-lifetime --steps 10 > gpurun_out/bench_cfg.json 2> gpurun_out/bench_cfg.err; python -c "
import json; j=json.loads(open('gpurun_out/bench_cfg.json').read().strip().splitlines()[-1])
print('value', j['value']/1e6, {k: round(v['value']/1e6,1) for k, v in j['other_configs'].items()})"
