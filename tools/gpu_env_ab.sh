# A/B of runtime knobs on the GPU box: bash tools/gpu_env_ab.sh "TW_PGS_TAIL=128" "TW_PGS_TAIL=512" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "$@"; do
    for rep in 1 2; do
        env $v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2> gpurun_out/ab.err
        python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
ph = d["resolve"]["phase_ms_count"]
keys = ["ph_refit", "ph_traverse", "ph_pgs_color", "ph_pgs_tail", "ph_color_conflict"]
print(f"{sys.argv[1]:>24} value {d['value']:.2f} kernel_ms {d['resolve']['kernel_ms']:.3f} " +
      " ".join(f"{k[3:]}={ph[k][0]:.3f}/{ph[k][1]}" for k in keys if k in ph))
PY
    done
done
