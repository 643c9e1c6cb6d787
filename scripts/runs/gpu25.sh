# NEXT-3 matrix-free measurements (C5 on one GPU, C2 fp32 product vs GEMV)
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python scripts/bench_configs.py C5_MF C2_MF > gpurun_out/configs_mf.json 2> gpurun_out/configs_mf.err; echo "rc=$?"
cat gpurun_out/configs_mf.json
