python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_mc.py tests/test_gpu_bem.py tests/test_gpu_geometry.py tests/test_gpu_poisson.py tests/test_gpu_mf.py tests/test_gpu_timer.py tests/test_gpu_galerkin.py tests/test_gpu_bm.py -q -x > gpurun_out/pt_b2.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_b2.log
