#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r02j}
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -3 gpurun_out/bench_$T.err
python -c "
import json; j=json.loads(open('gpurun_out/bench_$T.json').read().strip().splitlines()[-1])
print('value', j['value']/1e6, 'e2e', j['e2e']['value']/1e6, 'lifetime', j['lifetime']['value']/1e6, j['lifetime']['e2e']['value']/1e6)
print('roofline', json.dumps(j['roofline'])[:900])
print('dropin', {k: round(v['value']/1e6,1) for k, v in j['dropin_e2e'].items() if isinstance(v, dict)})
print('cpu', j.get('cpu_baseline'))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench2_$T.json 2> gpurun_out/bench2_$T.err
echo "rc=$?"; tail -c 1500 gpurun_out/bench2_$T.json; tail -5 gpurun_out/bench2_$T.err
