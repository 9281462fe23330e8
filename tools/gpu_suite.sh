#!/bin/bash
# Full GPU test suite + smoke (round-end style), results under gpurun_out/.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-suite}
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -s 2>&1 > gpurun_out/pytest_gpu_$T.full.log; echo "pytest rc=$?"
grep -E "passed|failed|error" gpurun_out/pytest_gpu_$T.full.log | tail -3
grep -E "loss .* vs ref|loss stair|hot-band|d512|text8 5 epochs|zipf|text8_d300|relative update error" gpurun_out/pytest_gpu_$T.full.log > gpurun_out/pytest_gpu_$T.quality.txt
tail -30 gpurun_out/pytest_gpu_$T.full.log > gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; tail -1 gpurun_out/smoke_$T.log
