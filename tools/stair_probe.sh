#!/bin/bash
# Staircase vs one-window wavefront: bitwise tests, then lifetime-order epochs (text8 d=128/d=300, 1bw d=128).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-stair}
timeout 900 python -m pytest tests/test_stair.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_stair_$TAG.log
tail -3 gpurun_out/pytest_stair_$TAG.log
for d in 128 300; do
  for ns in 0 1; do
    FW2V_NO_STAIR=$ns timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 10 --warmup 3 \
      --reuse-mode lifetime --dim $d 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('d=$d no_stair=$ns', round(j['value']/1e6,1), 'Mw/s')"
  done
done
