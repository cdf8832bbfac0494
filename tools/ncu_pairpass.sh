# ncu --set full of the standalone search and refresh kernels on the bow knot
# (tools/prof_search.py); prints time and the L1 traffic split (global vs local)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_stage_(search|refresh)' -c 2 \
  -o gpurun_out/prof_pairpass -f python tools/prof_search.py > gpurun_out/ncu_pairpass.log 2>&1
tail -2 gpurun_out/ncu_pairpass.log
