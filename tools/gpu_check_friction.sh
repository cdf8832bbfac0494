# Friction check: friction / dynamics tests, the bow-frame friction timing,
# then the bench line with extras (no cpu baseline).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_friction.py tests/test_gpu_dynamics.py -q -m gpu --timeout=600 -rf -x > gpurun_out/fric_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fric_tests.log
tail -6 gpurun_out/fric_tests.log
timeout 300 python tools/exp_friction.py > gpurun_out/exp_friction.log 2>&1; echo "exp rc=$?"; tail -3 gpurun_out/exp_friction.log
if [ "$1" = "bench" ]; then
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fric.log 2> gpurun_out/bench_fric.err; echo "bench rc=$?"
tail -c 300 gpurun_out/bench_fric.err
fi
