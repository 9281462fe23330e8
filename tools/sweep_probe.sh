#!/bin/bash
# BASELINE configs[4]-style sweep (text8 shape for speed): d x window x neg x reuse mode.
cd "$GRAFT_REPO_ROOT" || exit 1
for m in window_snapshot lifetime; do
  for a in "--dim 64" "--dim 256" "--dim 512" "--window 2" "--window 8" "--negatives 15" "--batch-sentences 1000" "--batch-sentences 50000"; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --reuse-mode $m $a 2>/dev/null | tail -1 | \
      python -c "import sys,json; j=json.loads(sys.stdin.read()); print('$m $a', round(j['value']/1e6,1), 'Mw/s frac', round(j['roofline']['frac'],3))" || echo "$m $a failed"
  done
done
