python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_mc.py tests/test_gpu_radiate.py --durations=6 2>&1 | tail -30
