#!/bin/bash
# BASELINE.json configs on one B200: text8 d=300 and the 1bw shape at d=128
# (text8 d=128 is bench.py's default line). SKIP_TESTS / SKIP_D300 / SKIP_1BW skip parts.
cd "$GRAFT_REPO_ROOT" || exit 1
summ() {
    python - "$1" "$2" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(j["value"] / 1e6, 1), "Mw/s  e2e", round(j["e2e"]["value"] / 1e6, 1),
          "frac", round(j["roofline"]["frac"], 3), "words/step", j["config"]["words_per_step_per_gpu"])
except Exception as e:  # noqa: BLE001
    print(sys.argv[1], "failed:", e)
PY
}
if [ -z "$SKIP_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2; fi
if [ -z "$SKIP_D300" ]; then
    timeout 300 python bench.py --no-cpu-baseline --steps 10 --dim 300 > gpurun_out/bench_d300.json 2> gpurun_out/bench_d300.err
    summ d300 gpurun_out/bench_d300.json
fi
if [ -z "$SKIP_1BW" ]; then
    start=$(date +%s)
    timeout 1500 python bench.py --no-cpu-baseline --steps 3 --workload 1bw > gpurun_out/bench_1bw.json 2> gpurun_out/bench_1bw.err
    echo "1bw wall $(( $(date +%s) - start )) s"; tail -3 gpurun_out/bench_1bw.err; free -g | head -2
    summ 1bw gpurun_out/bench_1bw.json
fi
