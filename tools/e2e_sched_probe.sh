#!/bin/bash
# e2e / device-resident scheduling knobs: kernel streams per lane, first short
# sub-batch, sub-batch target, chunk count.
cd "$GRAFT_REPO_ROOT" || exit 1
run() {
  env $1 timeout 300 python bench.py --no-cpu-baseline --steps 20 $2 2>&1 | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('$1 $2', round(j['value']/1e6,1), 'e2e', round(j['e2e']['value']/1e6,1), flush=True)"
}
run "FW2V_KSTREAMS=1" "--chunks 64"
run "FW2V_KSTREAMS=2" "--chunks 64"
run "FW2V_KSTREAMS=2 FW2V_FIRST_SUB=0" "--chunks 64"
run "FW2V_KSTREAMS=2 FW2V_SUB_TARGET=128" "--chunks 64"
run "FW2V_KSTREAMS=2 FW2V_SUB_TARGET=64" "--chunks 64"
run "FW2V_KSTREAMS=2" "--chunks 128"
run "FW2V_KSTREAMS=2 FW2V_SUB_TARGET=128" "--chunks 32"
run "FW2V_KSTREAMS=2" "--chunks 64 --reuse-mode lifetime"
run "FW2V_KSTREAMS=1" "--chunks 64 --reuse-mode lifetime"
