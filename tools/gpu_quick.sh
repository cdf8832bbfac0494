cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout=300 -rf -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
grep -E "passed|failed|Error|assert" gpurun_out/gpu_tests.log | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "kernel_ms", d["resolve"]["kernel_ms"], "frac", d["roofline"]["frac"])
print({k: v for k, v in d["resolve"]["phase_ms_count"].items()})
PY
tail -3 gpurun_out/bench.err
