# fp64 far kernel with 4-row CTAs, warp-per-row matrix-free epilogue: parity + measurements + ncu
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1200 python -m pytest tests/test_gpu_mf.py tests/test_gpu_bem.py tests/test_gpu_configs.py tests/test_gpu_bm.py -x -q > gpurun_out/pytest_27.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_27.log
timeout 900 python scripts/bench_configs.py C5_MF C2_MF C5 > gpurun_out/configs_27.json 2> gpurun_out/configs_27.err; echo "cfg rc=$?"
cat gpurun_out/configs_27.json
ncu --set full --clock-control none --import-source on -k regex:"far_kernel|mf_final" -c 6 \
    -o /tmp/prof_mf python scripts/prof_mf.py > gpurun_out/ncu_mf27.log 2>&1
echo "ncu rc=$?"
python scripts/summarize_ncu.py /tmp/prof_mf.ncu-rep > gpurun_out/prof_mf27_summary.md
python scripts/stalls.py /tmp/prof_mf.ncu-rep > gpurun_out/prof_mf27_stalls.txt
cat gpurun_out/prof_mf27_summary.md gpurun_out/prof_mf27_stalls.txt
