#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for rep in 1 2; do for v in old ""; do
  L=""; [ -n "$v" ] && L=$PWD/paper_2312_07743_b200/_lib/libfw2v_$v.so
  FW2V_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode lifetime 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lifetime d=128 W=5 lib [$v]', round(j['value']/1e6,1), 'Mw/s', j['clocks']['reasons'])"
done; done
python tools/e2e_gap_probe.py 2>&1 | tail -6
timeout 600 python -m pytest tests/test_quality.py -q -x -k "d512" 2>&1 | tail -2
