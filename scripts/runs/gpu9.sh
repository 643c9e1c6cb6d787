python -m paper_2506_06190_b200.build > /dev/null || exit 1
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"far_kernel_x2|near_kernel" -c 8 \
    -o gpurun_out/prof_r01b python scripts/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
