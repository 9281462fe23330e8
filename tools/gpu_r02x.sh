#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for m in window_snapshot lifetime; do for hm in 1 0; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode $m --hot-merge $hm 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m hot_merge=$hm', round(j['value']/1e6,1), 'Mw/s')"
done; done
timeout 1500 python -m pytest tests/test_quality.py -q -s -k "text8" 2>&1 | grep -E "text8|passed|failed"
