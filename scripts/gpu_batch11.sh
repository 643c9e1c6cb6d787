python -m paper_2506_06190_b200.build > /dev/null || exit 1
for r in 1 2 3; do timeout 600 python bench.py --steps 3 --warmup 2 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_v$r.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_v$r.json'));print('rep',$r,round(d['value'],1),round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
for w in 2 3; do timeout 600 python bench.py --steps 3 --warmup 2 --workers $w --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_w$w.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_w$w.json'));print('workers',$w,round(d['value'],1),round(d['ms_per_step'],1))"; done
