#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for args in "--reuse-mode lifetime --k1-lanes 32" "--reuse-mode window_snapshot --k1-lanes 32" "--reuse-mode lifetime --hot-rows 0" "--reuse-mode lifetime --l1-refresh-log2 0"; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 $args 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$args', round(j['value']/1e6,1), 'Mw/s')"
done
