#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/dropin_probe.py > gpurun_out/dropin_probe_r02b.txt 2>&1
tail -30 gpurun_out/dropin_probe_r02b.txt
bash tools/stair_probe.sh r02b
