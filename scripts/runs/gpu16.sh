python -m paper_2506_06190_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"radiate_f32x2_kernel|far_kernel_x2|gemv_c64_kernel|near_kernel<float" -c 9 \
    -o gpurun_out/prof_r01_full python scripts/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
