python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_radiate.py tests/test_gpu_mc.py tests/test_gpu_configs.py -q -x > gpurun_out/pt_b12.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_b12.log
for a in 1 0; do if [ $a = 0 ]; then export NAT_NO_ARITH=1; fi; echo "arith $a"; timeout 300 python scripts/prof_c4.py 0 2 2>&1 | tail -1; timeout 600 python bench.py --steps 3 --warmup 2 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_a$a.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_a$a.json'));print('arith',$a,round(d['value'],1),round(d['ms_per_step'],1));[print(k,round(v['frac'],3),round(v['achieved'])) for k,v in d['rooflines'].items()]"; done
