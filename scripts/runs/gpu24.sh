# Matrix-free dense operator (NEXT-3): GPU parity tests.
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1200 python -m pytest tests/test_gpu_mf.py -x -q --durations=10 > gpurun_out/pytest_mf.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_mf.log
