# A/B of compile-time variants on the GPU box: bash tools/gpu_ab.sh "-DX=1" "-DX=2" ...
# Rebuilds the library per variant (nvcc is in the image) and runs a short bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "$@"; do
    rm -f build/tw_kernels.o build/tw_capi.o
    make -s NVEXTRA="$v" > gpurun_out/ab_build.log 2>&1 || { echo "build failed: $v"; tail gpurun_out/ab_build.log; continue; }
    for rep in 1 2; do
        timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2> gpurun_out/ab.err
        python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
ph = d["resolve"]["phase_ms_count"]
keys = ["ph_traverse", "ph_cand_eval", "ph_emit_records", "ph_refresh", "ph_pgs_color", "ph_rows"]
print(f"{sys.argv[1]:>24} value {d['value']:.2f} kernel_ms {d['resolve']['kernel_ms']:.3f} " +
      " ".join(f"{k[3:]}={ph[k][0]:.3f}" for k in keys if k in ph))
PY
    done
done
