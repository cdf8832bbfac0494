# A/B of two builds of the library on the bench frame: $1 = A .so (TW_LIB_PATH),
# B = the default in-tree build; alternated 3 times, plus the parity tests on B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py tests/test_gpu_large.py tests/test_gpu_configs.py -q -m gpu --timeout=600 -x > gpurun_out/ab_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab_tests.log
for r in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then export TW_LIB_PATH=$GRAFT_REPO_ROOT/$1; else unset TW_LIB_PATH; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ab.log 2>&1
    python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
ph = d["resolve"]["phase_ms_count"]
print(sys.argv[1], "value", d["value"], "resolve", round(d["frame"]["resolve_ms"], 3), "pcg", round(d["frame"]["pcg_ms"], 3),
      {k: round(ph[k][0], 3) for k in ("ph_refresh", "ph_emit_records", "ph_cand_eval", "ph_traverse") if k in ph})
PY
  done
done
