python -m paper_2506_06190_b200.build > /dev/null || exit 1
python scripts/prof_kernels.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"far_kernel_x2|near_kernel|mc_finish|cdf_kernel|scan_i32" -c 8 \
    -o gpurun_out/prof_far python scripts/prof_kernels.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
python scripts/summarize_ncu.py gpurun_out/prof_far.ncu-rep > gpurun_out/prof_far_summary.md
python scripts/stalls.py gpurun_out/prof_far.ncu-rep > gpurun_out/prof_far_stalls.txt
ncu -i gpurun_out/prof_far.ncu-rep --page source --csv -k regex:far_kernel_x2 > gpurun_out/prof_far_source.csv 2>/dev/null
ls -la gpurun_out/prof_far*
