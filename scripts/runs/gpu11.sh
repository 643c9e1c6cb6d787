python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest -x -q -m gpu tests/ 2>&1 | tail -3
python scripts/quick_rad.py 2>&1 | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"
python - <<'P'
import json; d=json.load(open('gpurun_out/bench5.json'))
print(d['value'], d['ms_per_step'], d['phase_ms_per_step'], d['gmres_iters'], d['mc_gmres_iters'])
for k,v in d['rooflines'].items(): print(k, round(v['achieved'],1), round(v['frac'],3))
print(d['clocks'])
P
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile-count > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
