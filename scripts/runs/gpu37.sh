# Krylov finish tail + 16-vector update batches: GMRES parity + bench phases + warm launch list
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_bem.py tests/test_gpu_mc.py tests/test_gpu_mf.py -x -q > gpurun_out/pytest_37.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_37.log
for rep in 1 2; do
python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/b37.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b37.json'))
r=d['rooflines']; print(round(d['value'],1), round(d['ms_per_step'],2), {k:round(v,3) for k,v in d['phase_ms_per_step'].items()})"
done
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count --no-overlap > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm37.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count --no-overlap > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_warm37.csv 4 | head -16
