cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/prof_search.py > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 1 -c 2 -o gpurun_out/prof_search python tools/prof_search.py > gpurun_out/ncu_search.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_search.log; cat gpurun_out/plain2.log
