#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for rep in 1 2; do for m in lifetime window_snapshot; do for v in "" sat snap7; do
  L=""; [ -n "$v" ] && L=$PWD/paper_2312_07743_b200/_lib/libfw2v_$v.so
  FW2V_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-dropin --no-lifetime --steps 20 --warmup 3 --reuse-mode $m 2>/dev/null | python -c "import sys,json; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m lib [$v]', round(j['value']/1e6,1), 'Mw/s')"
done; done; done
FW2V_LIB=$PWD/paper_2312_07743_b200/_lib/libfw2v_sat.so timeout 900 python -m pytest tests/test_stair.py tests/test_parity_bench.py -q -x -k "128" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_quality.py -q -s -k "other_shapes" 2>&1 | grep -E "zipf|d300|passed|failed"
