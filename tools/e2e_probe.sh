#!/bin/bash
# e2e (C-ABI, host batching) vs device-resident value for a few host settings.
cd "$GRAFT_REPO_ROOT" || exit 1
for a in "--chunks 64" "--chunks 32" "--chunks 64 --streams 12"; do
  timeout 300 python bench.py --no-cpu-baseline --steps 20 $a 2>&1 | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('$a', round(j['value']/1e6,1), 'e2e', round(j['e2e']['value']/1e6,1), 'batch/thread', round(j['e2e']['host_batching_words_per_sec_per_thread']/1e6,1))"
done
CHUNKS=64 python tools/e2e_trace.py 2> gpurun_out/trace64.txt | tail -2
