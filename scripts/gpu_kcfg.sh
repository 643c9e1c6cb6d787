python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_bench_sweep.py tests/test_gpu_multirank.py -q -x 2>&1 | tail -1
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 $B 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1), {k: round(v['frac'],3) for k,v in d['rooflines'].items()})
s=d['secondary']; print({k: (round(s[k].get('value') or 0,1), round(s[k]['ms_per_step'],3)) for k in ('C2','C3','NEXT4')})"
