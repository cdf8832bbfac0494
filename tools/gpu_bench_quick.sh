# quick GPU pass: dynamics tests + a short bench line (no cpu baseline)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dynamics.py -q -m gpu --timeout=600 -x > gpurun_out/gpu_dyn.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_dyn.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_q.log 2> gpurun_out/bench_q.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.log").read().strip().splitlines()[-1])
for k in ("value", "ms_per_step", "gpu_launches"):
    print(k, d.get(k))
print("e2e", d["e2e"]["value"])
print("frame", d["frame"])
print("roofline", {k: d["roofline"][k] for k in ("achieved", "frac")}, d["roofline"]["pcg"])
print("resolve", {k: d["resolve"][k] for k in ("alg1_steps", "searches", "kernel_ms", "setup_ms")})
print("ccd", d["ccd_certification"])
for k in ("resolve_only", "exact_parity_mode", "batch_configs4_one_gpu"):
    print(k, d.get(k))
print({k: v for k, v in d["resolve"]["phase_ms_count"].items()})
PY
