# Krylov kernel change: GMRES/MC parity tests, then a warm-cache launch list of the bench step.
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_bem.py tests/test_gpu_mc.py -x -q > gpurun_out/pytest_23.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_23.log
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count --no-overlap > gpurun_out/plain23.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count --no-overlap > gpurun_out/ncu23.log 2>&1
echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/launches_warm.csv 4 > gpurun_out/launches_warm_summary.txt
head -30 gpurun_out/launches_warm_summary.txt
