#!/bin/bash
# Round-end evidence: GPU suite + smoke, bench (ours, reference arm), 2 ranks on 1 GPU.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r02final}
bash tools/gpu_suite.sh $T
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -2 gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; tail -c 600 gpurun_out/bench_ref_$T.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench2_$T.json 2> gpurun_out/bench2_$T.err; echo "2-rank rc=$?"
python -c "
import json; j=json.loads(open('gpurun_out/bench_$T.json').read().strip().splitlines()[-1])
print('value', j['value']/1e6, 'e2e', j['e2e']['value']/1e6, 'lifetime', j['lifetime']['value']/1e6, j['lifetime']['e2e']['value']/1e6)
print('dropin', {k: round(v['value']/1e6,1) for k, v in j['dropin_e2e'].items() if isinstance(v, dict)})
print('clocks', j['clocks'], 'roofline', round(j['roofline']['frac'],3), round(j['roofline']['l2']['frac'],3))"
