#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/e2e_gap_probe.py > gpurun_out/e2e_gap.txt 2>&1; cat gpurun_out/e2e_gap.txt
FW2V_TRACE=1 python tools/e2e_gap_probe.py > /dev/null 2> gpurun_out/e2e_trace.txt; wc -l gpurun_out/e2e_trace.txt
