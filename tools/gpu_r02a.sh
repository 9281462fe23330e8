cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r02a.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -40 > gpurun_out/pytest_gpu_r02a.log
tail -5 gpurun_out/pytest_gpu_r02a.log
timeout 600 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
tail -c 3000 gpurun_out/bench_r02a.json; tail -5 gpurun_out/bench_r02a.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02a.log 2>&1; tail -2 gpurun_out/smoke_r02a.log
