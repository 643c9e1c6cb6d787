python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for cl in 8 4; do echo "CL $cl"; NAT_FUSED_CL=$cl timeout 300 python scripts/prof_c4.py 0 2 2>&1 | tail -1; NAT_FUSED_CL=$cl timeout 300 python -m pytest tests/test_gpu_mc.py -q -x -k "surface_pressure" 2>&1 | tail -1; done
for cl in 8 4; do NAT_FUSED_CL=$cl timeout 600 python bench.py --steps 3 --warmup 2 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_cl$cl.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_cl$cl.json'));print('CL',$cl,round(d['value'],1),round(d['ms_per_step'],1))"; done
