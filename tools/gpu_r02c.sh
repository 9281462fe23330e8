#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
FW2V_TRACE=1 timeout 300 python tools/dropin_trace.py dropin > gpurun_out/trace_dropin.txt 2>&1
FW2V_TRACE=1 timeout 300 python tools/dropin_trace.py corpus > gpurun_out/trace_corpus.txt 2>&1
wc -l gpurun_out/trace_*.txt
