#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_stair.py tests/test_observer.py -q -x 2>&1 | tail -1
for m in lifetime window_snapshot; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode $m 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(j['value']/1e6,1), 'Mw/s')"
done
bash tools/final_profiles.sh r02cc lifetime > /dev/null 2>&1; head -14 gpurun_out/quick_lifetime_r02cc.txt; rm -f gpurun_out/*.ncu-rep
