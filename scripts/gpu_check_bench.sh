python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_bench_sweep.py -q -x > gpurun_out/pt_b39.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_b39.log
NAT_BENCH_VERBOSE=1 timeout 1500 python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_b39.json 2> gpurun_out/bench_b39.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_b39.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['mc_gmres_iters'])
for k,v in d['rooflines'].items(): print(k, round(v['frac'],3), v['seconds'])
print(d['roofline']['dominant'], d['roofline']['share_of_serialised_step'])
PY
