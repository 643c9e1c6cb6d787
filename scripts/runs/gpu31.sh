# Galerkin near kernel rework: parity + measurement + ncu
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_galerkin.py -x -q > gpurun_out/pytest_gal31.log 2>&1; echo "pytest gal rc=$?"
tail -3 gpurun_out/pytest_gal31.log
timeout 600 python scripts/bench_configs.py GAL_C2 > gpurun_out/configs_gal31.json 2> gpurun_out/configs_gal31.err; echo "cfg rc=$?"
cat gpurun_out/configs_gal31.json
python scripts/prof_gal.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"far_kernel|gal_" -c 4 \
    -o /tmp/prof_gal python scripts/prof_gal.py > gpurun_out/ncu_gal31.log 2>&1
echo "ncu rc=$?"
python scripts/summarize_ncu.py /tmp/prof_gal.ncu-rep > gpurun_out/prof_gal31_summary.md
python scripts/stalls.py /tmp/prof_gal.ncu-rep > gpurun_out/prof_gal31_stalls.txt
cat gpurun_out/prof_gal31_summary.md gpurun_out/prof_gal31_stalls.txt
