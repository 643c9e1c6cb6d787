# NEXT-2 Galerkin: GPU parity tests (+ collocation regressions of the modified far kernels)
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_galerkin.py -x -q --durations=8 > gpurun_out/pytest_gal.log 2>&1; echo "pytest gal rc=$?"
tail -30 gpurun_out/pytest_gal.log
timeout 900 python -m pytest tests/test_gpu_bem.py tests/test_gpu_bm.py tests/test_gpu_mf.py -x -q > gpurun_out/pytest_reg.log 2>&1; echo "pytest reg rc=$?"
tail -3 gpurun_out/pytest_reg.log
