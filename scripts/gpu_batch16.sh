python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_bem.py -q -x -k "multi" > gpurun_out/pt_b16.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_b16.log
timeout 300 python scripts/c2_far_multi.py 2>&1 | tail -2
