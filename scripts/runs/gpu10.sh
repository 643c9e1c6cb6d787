python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_bem.py 2>&1 | tail -2
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
