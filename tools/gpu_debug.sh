cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export TW_DEBUG=1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_dbg.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_dbg.log
tail -3 gpurun_out/smoke_dbg.log
