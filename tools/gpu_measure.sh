# Round measurement pass: default bench line (with cpu_baseline), the reference
# arm, the ncu launch list of the bench command, and --set full captures of the
# frame's resolve kernel, its CG kernel and the search stage. Each ncu pass
# only after the same command exited 0 without ncu.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(time timeout 900 ./oracle/_ref/b200/acceptance_groups 1_2_6 3 4 10 11) > gpurun_out/acc_b200.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -c 400 gpurun_out/bench_full.log
timeout 1800 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -c 600 gpurun_out/bench_ref.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/b2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
timeout 300 python tools/prof_drive.py > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_resolve|k_pcg_reg" -c 2 \
    -o gpurun_out/prof_resolve -f python tools/prof_drive.py > gpurun_out/ncu_full.log 2>&1
echo "ncu frame rc=$?"; tail -2 gpurun_out/ncu_full.log
timeout 300 python tools/prof_search.py > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_stage -c 2 \
    -o gpurun_out/prof_search -f python tools/prof_search.py > gpurun_out/ncu_search.log 2>&1
echo "ncu search rc=$?"; tail -2 gpurun_out/ncu_search.log
# Summarise on the box (the .ncu-rep files exceed gpurun's 64 MiB merge limit):
# profiles are staged under gpurun_out/profiles_staged and copied into
# profiles/ here; the reports are then removed from gpurun_out.
TW_PROF_DIR=gpurun_out/profiles_staged python tools/make_profiles.py ${PROF_TAG:-r02} > gpurun_out/make_profiles.log 2>&1
echo "make_profiles rc=$?"; tail -2 gpurun_out/make_profiles.log
rm -f gpurun_out/*.ncu-rep
