# fp64 fast sincos: fp64 parity tests + C5 measurements
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_mf.py tests/test_gpu_bem.py tests/test_gpu_radiate.py tests/test_gpu_configs.py tests/test_gpu_galerkin.py tests/test_gpu_mc.py -x -q > gpurun_out/pytest_32.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_32.log
timeout 900 python scripts/bench_configs.py C5_MF C5 > gpurun_out/configs_32.json 2> gpurun_out/configs_32.err; echo "cfg rc=$?"
cat gpurun_out/configs_32.json
