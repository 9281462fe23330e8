#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_stair.py -q -k bitwise 2>&1 | grep -E "^FAILED|passed|failed" | head -20
for d in 64 128 256 300; do for w in 8 10; do for v in base ""; do
  L=""; [ -n "$v" ] && L=$PWD/paper_2312_07743_b200/_lib/libfw2v_$v.so
  FW2V_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 8 --warmup 3 --reuse-mode lifetime --window $w --dim $d 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lifetime d=$d W=$w lib [$v]', round(j['value']/1e6,1), 'Mw/s')"
done; done; done
