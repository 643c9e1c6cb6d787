python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_multirank.py tests/test_gpu_configs.py -q -x > gpurun_out/pt_b28.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_b28.log
bash scripts/gpu_batch27.sh 2>&1 | tail -1
echo "== default"; timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -2
