# Round-end check: every GPU test, smoke, and the default bench line
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])
s=d['secondary']; print({k: (round(s[k].get('value') or 0,1), round(s[k]['ms_per_step'],3)) for k in ('C2','C3','NEXT4')})
PY
