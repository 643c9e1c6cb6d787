# Round profile refresh (run under gpurun): bench line, launch list, ncu --set full of the
# hot kernels, stall reasons, per-config measurements.  Outputs in gpurun_out/; copy the
# summaries to profiles/.
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
# launch list of one serialised step: 3 warm-up + 1 timed + 1 kernel-timer step => divide by 5
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count --no-overlap > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count --no-overlap > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/launches.csv 5 > gpurun_out/launches_summary.txt
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"far_kernel_x2|radiate_f32x2|gemv_c64|mc_finish|near_kernel|dots_kernel|update_kernel|stage_kernel" \
    -c 60 -o /tmp/prof_full python scripts/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
python scripts/summarize_ncu.py /tmp/prof_full.ncu-rep gpurun_out/traffic.json > gpurun_out/ncu_full_summary.md
python scripts/stalls.py /tmp/prof_full.ncu-rep > gpurun_out/ncu_full_stalls.txt
timeout 1500 python scripts/bench_configs.py > gpurun_out/configs_all.json 2> gpurun_out/configs_all.err; echo "configs rc=$?"
ls -la gpurun_out/; du -sh gpurun_out
