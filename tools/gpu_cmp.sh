cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout=300 -rf -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
grep -E "passed|failed|Error" gpurun_out/gpu_tests.log | tail -3
for b in 2 3 4; do
  TW_BLOCKS_PER_SM=$b timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b$b.log 2> gpurun_out/bench_b$b.err
  python - "$b" <<'PY'
import json, sys
b = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_b{b}.log").read().strip().splitlines()[-1])
print("blocks/SM", b, "value", d["value"], "kernel_ms", d["resolve"]["kernel_ms"], {k: v[0] for k, v in d["resolve"]["phase_ms_count"].items()})
PY
done
