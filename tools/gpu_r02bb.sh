#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for rep in 1 2; do for v in "" rb5 rb6; do
  L=""; [ -n "$v" ] && L=$PWD/paper_2312_07743_b200/_lib/libfw2v_$v.so
  FW2V_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode lifetime 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lifetime lib [$v]', round(j['value']/1e6,1), 'Mw/s')"
done; done
