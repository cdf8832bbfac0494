# A/B of env settings on the bench frame: prints value and the main phases per variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "$@"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ab.log 2>&1
  python - "$v" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", open("gpurun_out/ab.log").read()[-300:]); sys.exit()
ph = d["resolve"]["phase_ms_count"]
top = sorted(ph.items(), key=lambda kv: -kv[1][0])[:8]
print(sys.argv[1], "value", d["value"], "frame", d["frame"]["ms"], "resolve", d["frame"]["resolve_ms"], "pcg", d["frame"]["pcg_ms"],
      {k: v[0] for k, v in top})
PY
done
