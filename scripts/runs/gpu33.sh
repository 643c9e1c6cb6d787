# kernel-timer rooflines in bench.py
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python bench.py > gpurun_out/bench_33.json 2> gpurun_out/bench_33.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_33.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'])
print('ROOFLINE', json.dumps(d['roofline']))
for k,v in d['rooflines'].items(): print(k, round(v.get('frac',0),3), v.get('achieved'), v.get('ms_per_step'), v.get('launches_per_step'))
"
tail -5 gpurun_out/bench_33.err
