# ncu --set full of the friction replay kernel on the bow frame (tools/exp_friction.py),
# summarised on the box into gpurun_out/r02_ncu_friction.txt (the report is removed).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/exp_friction.py > gpurun_out/fr_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_friction|k_fr_eval0|k_fr_verify" -c 3 \
    -o gpurun_out/prof_fr -f python tools/exp_friction.py > gpurun_out/ncu_fr.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_fr.log
python - <<'PY'
import sys
sys.path.insert(0, "tools")
import make_profiles as M
out = [M.summarize("gpurun_out/prof_fr.ncu-rep", "k_friction",
                   "friction_filter on the bow frame (tools/exp_friction.py): k_fr_eval0 (every pair at y0), "
                   "k_friction (the replay over W, round 0), k_fr_verify")[0]]
open("gpurun_out/r02_ncu_friction.txt", "w").write("\n".join(out))
print("summary written")
PY
rm -f gpurun_out/prof_fr.ncu-rep
