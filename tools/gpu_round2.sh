#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r02r}
bash tools/gpu_suite.sh $T
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -3 gpurun_out/bench_$T.err
python -c "
import json; j=json.loads(open('gpurun_out/bench_$T.json').read().strip().splitlines()[-1])
print('value', j['value']/1e6, 'e2e', j['e2e']['value']/1e6, 'lifetime', j['lifetime']['value']/1e6, j['lifetime']['e2e']['value']/1e6)
print('dropin', {k: round(v['value']/1e6,1) for k, v in j['dropin_e2e'].items() if isinstance(v, dict)})
print('clocks', j['clocks'])"
