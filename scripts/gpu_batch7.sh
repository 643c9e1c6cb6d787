python -m paper_2506_06190_b200.build > /dev/null || exit 1
for f in 1 0; do for w in 4 6; do NAT_GMRES_FUSED=$f timeout 600 python bench.py --steps 2 --warmup 1 --workers $w --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_f${f}_w$w.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_f${f}_w$w.json'));print('fused',$f,'workers',$w,round(d['value'],1),round(d['ms_per_step'],1))"; done; done
