cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export TW_DEBUG=1
timeout 600 python tools/gpu_diag.py > gpurun_out/diag.log 2>&1; echo "rc=$?" >> gpurun_out/diag.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "battery or pymodule" > gpurun_out/diag2.log 2>&1; echo "rc=$?" >> gpurun_out/diag2.log
tail -20 gpurun_out/diag.log; grep -E "Error|progress|passed|failed" gpurun_out/diag2.log | tail
