cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for t in 0 256 1024 4096; do
  TW_PGS_TAIL=$t timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tail_$t.log 2>&1
  python - $t <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/tail_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("tail", sys.argv[1], "value", d["value"], "kernel_ms", d["resolve"]["kernel_ms"])
PY
done
