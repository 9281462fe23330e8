#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r02d}
timeout 900 python -m pytest tests/test_stair.py tests/test_guard.py tests/test_parity_bench.py tests/test_gpu_parity.py -x -q 2>&1 | tail -8 > gpurun_out/pytest_$T.log; tail -3 gpurun_out/pytest_$T.log
timeout 600 python tools/dropin_probe.py > gpurun_out/dropin_probe_$T.txt 2>&1; cat gpurun_out/dropin_probe_$T.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; python -c "
import json; j=json.loads(open('gpurun_out/bench_$T.json').read().strip().splitlines()[-1])
print('value', j['value']/1e6, 'e2e', j['e2e']['value']/1e6, 'lifetime', j['lifetime']['value']/1e6, j['lifetime']['e2e']['value']/1e6)
print('dropin', json.dumps(j.get('dropin_e2e'))[:600])"
