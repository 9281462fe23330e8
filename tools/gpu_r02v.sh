#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for rep in 1 2; do for m in window_snapshot lifetime; do for v in "" l2; do
  L=""; [ -n "$v" ] && L=$PWD/paper_2312_07743_b200/_lib/libfw2v_$v.so
  for l1 in 5 0; do
  FW2V_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode $m --l1-refresh-log2 $l1 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m l1_refresh_log2=$l1 lib [$v]', round(j['value']/1e6,1), 'Mw/s')"
  done
done; done; done
