python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_radiate.py tests/test_gpu_mc.py -q -x > gpurun_out/pt_b6.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_b6.log
for mb in 4 8; do echo "MB cap $mb"; NAT_MAX_MB=$mb NAT_DEBUG_PLAN=1 timeout 300 python scripts/prof_c4.py 0 2 > gpurun_out/c4_mb$mb.log 2>&1; tail -1 gpurun_out/c4_mb$mb.log; grep "kind 0 modes 64\|kind 1 modes 64 " gpurun_out/c4_mb$mb.log | sort | uniq | head -3; done
for mb in 4 8; do NAT_MAX_MB=$mb timeout 600 python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_mb$mb.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_mb$mb.json'));print('MB',$mb,d['value'],d['ms_per_step']);[print(k,round(v['frac'],3),round(v['achieved'])) for k,v in d['rooflines'].items()]"; done
