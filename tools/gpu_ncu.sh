cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
sed -n '/prof_drive.py > gpurun_out\/plain.log/,$p' tools/gpu_measure.sh > /tmp/ncu_part.sh
bash /tmp/ncu_part.sh
