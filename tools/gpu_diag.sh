cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/gpu_diag.py > gpurun_out/diag.log 2>&1; echo "rc=$?" >> gpurun_out/diag.log
tail -20 gpurun_out/diag.log
