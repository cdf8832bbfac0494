cd $GRAFT_REPO_ROOT
for mb in ${@:-4 3 2}; do
  TW_REFRESH_MINB=$mb timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_stage_refresh --csv python tools/prof_search.py 2>/dev/null | grep -E "gpu__time|warps_active" | awk -F'","' -v mb=$mb '{print mb, $(NF-2), $NF}'
done
