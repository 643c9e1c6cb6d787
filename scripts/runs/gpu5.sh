python -m paper_2506_06190_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
# launch list of one bench step (after 3 warm-up steps): per-launch device times
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
# full capture of the hot kernels (second repetition of each)
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"radiate_f32_kernel|far_kernel|near_kernel|gemv_c64_kernel|self_kernel" -c 12 \
    -o gpurun_out/prof_r01 python scripts/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
