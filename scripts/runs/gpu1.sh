set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2506_06190_b200.build
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_geometry.py tests/test_gpu_radiate.py 2>&1 | tail -30
timeout 300 python scripts/quick_rad.py
