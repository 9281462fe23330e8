#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for l1 in 5 0; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode lifetime --l1-refresh-log2 $l1 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lifetime l1=$l1', round(j['value']/1e6,1), 'Mw/s')"
done
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode lifetime --dim 300 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lifetime d=300', round(j['value']/1e6,1), 'Mw/s')"
timeout 900 python -m pytest tests/test_stair.py tests/test_parity_bench.py -q -x -k "stair or lifetime" 2>&1 | tail -2
