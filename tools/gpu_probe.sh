cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python tools/scene_probe.py > gpurun_out/probe.log 2>&1; echo "rc=$?" >> gpurun_out/probe.log
cat gpurun_out/probe.log | tail -12
