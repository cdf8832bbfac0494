cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/bench.log; tail -5 gpurun_out/bench.err
