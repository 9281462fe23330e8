#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_stair.py tests/test_gpu_parity.py tests/test_observer.py -q -x -s -k "n15 or hot_replicas or bitwise or observer" 2>&1 | grep -E "N=15|passed|failed|FAILED|Error" | tail -8
for n in 15 5; do for ns in 0 1; do
FW2V_NO_STAIR=$ns timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 10 --warmup 3 --reuse-mode lifetime --negatives $n 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lifetime N=$n no_stair=$ns', round(j['value']/1e6,1), 'Mw/s')"
done; done
