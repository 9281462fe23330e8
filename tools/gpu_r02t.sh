#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for m in window_snapshot lifetime; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode $m 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(j['value']/1e6,1), 'Mw/s', j['clocks']['reasons'])"
done
timeout 900 python -m pytest tests/test_observer.py tests/test_stair.py tests/test_guard.py -q -x 2>&1 | tail -2
python tools/e2e_gap_probe.py 2>&1 | grep "10-epoch"
