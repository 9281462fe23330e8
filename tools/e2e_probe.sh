cd $GRAFT_REPO_ROOT
grep -i AnonHugePages /proc/meminfo; cat /sys/kernel/mm/transparent_hugepage/enabled
for smp in reference alias; do
  timeout 300 python bench.py --no-cpu-baseline --steps 20 --sampler $smp 2>&1 | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('$smp', round(j['value']/1e6,1), 'e2e', round(j['e2e']['value']/1e6,1), 'batch/thread', round(j['e2e']['host_batching_words_per_sec_per_thread']/1e6,1))"
done
for st in 8 32; do
  timeout 300 python bench.py --no-cpu-baseline --steps 20 --streams $st --sampler alias 2>&1 | tail -1 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('streams $st', round(j['value']/1e6,1), 'e2e', round(j['e2e']['value']/1e6,1), 'batch/thread', round(j['e2e']['host_batching_words_per_sec_per_thread']/1e6,1))"
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
