# pipe-rate ubench (DFMA, MUFU.RSQ added) + ncu full of the matrix-free far kernels
python -m paper_2506_06190_b200.build > /dev/null || exit 1
./scripts/ubench_pipes > gpurun_out/ubench26.txt 2>&1; cat gpurun_out/ubench26.txt
python scripts/prof_mf.py > gpurun_out/prof_mf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"far_kernel|mf_final" -c 6 \
    -o /tmp/prof_mf python scripts/prof_mf.py > gpurun_out/ncu_mf.log 2>&1
echo "ncu rc=$?"
python scripts/summarize_ncu.py /tmp/prof_mf.ncu-rep > gpurun_out/prof_mf_summary.md
python scripts/stalls.py /tmp/prof_mf.ncu-rep > gpurun_out/prof_mf_stalls.txt
cp /tmp/prof_mf.ncu-rep gpurun_out/ 2>/dev/null
cat gpurun_out/prof_mf_summary.md gpurun_out/prof_mf_stalls.txt
