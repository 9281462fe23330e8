#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for v in "" wf4; do
  L=""; [ -n "$v" ] && L=$PWD/paper_2312_07743_b200/_lib/libfw2v_$v.so
  FW2V_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 10 --warmup 3 --reuse-mode lifetime --window 8 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lifetime W=8 variant [$v]', round(j['value']/1e6,1), 'Mw/s')"
done
FW2V_LIB=$PWD/paper_2312_07743_b200/_lib/libfw2v_wf4.so timeout 600 python -m pytest tests/test_stair.py -x -q -k "bitwise and 128" 2>&1 | tail -1
