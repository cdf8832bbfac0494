# GPU test pass: the parity suite (or a subset: $1 = pytest -k / path args)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest ${@:-tests} -q -m gpu --timeout=600 -rf -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -25 gpurun_out/gpu_tests.log
