python -m paper_2506_06190_b200.build > /dev/null || exit 1
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"far_kernel_x2|radiate_f32x2|mc_finish|update_kernel|dots_kernel|gemv_c64" -s 12 -c 14 \
    -o gpurun_out/prof_r2 python scripts/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
python scripts/summarize_ncu.py gpurun_out/prof_r2.ncu-rep > gpurun_out/prof_r2_summary.md
python scripts/stalls.py gpurun_out/prof_r2.ncu-rep > gpurun_out/prof_r2_stalls.txt
