python -m paper_2506_06190_b200.build > /dev/null || exit 1
for cfg in "120 0" "0 0" "0 1" "120 1"; do set -- $cfg; export NAT_FUSED_SMEM_KB=$1 NAT_FUSED_NARROW=$2
timeout 600 python bench.py --steps 3 --warmup 2 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_f.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_f.json'));print('smem $1 narrow $2',round(d['value'],1),round(d['ms_per_step'],1))"; done
