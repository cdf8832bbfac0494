cd $GRAFT_REPO_ROOT
for s in 0 64 256 1024; do TW_FLOW_SLEEP=$s python tools/exp_search.py | grep -E "kernel_ms|pgs"; done
TW_PGS_FLOW=0 python tools/exp_search.py | grep -E "kernel_ms|pgs"
