cd $GRAFT_REPO_ROOT
for t in 0 64 128 256 512; do echo "tail=$t"; TW_PGS_TAIL=$t python tools/exp_steps.py ph_pgs_color ph_pgs_tail | tail -1; done
