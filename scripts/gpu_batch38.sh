python -m paper_2506_06190_b200.build > /dev/null || exit 1
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
run() { echo "== $1"; env NAT_BENCH_VERBOSE=1 $1 timeout 600 $B 2>&1 | grep -E "step ms|^\{" | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(round(d['value'],1), round(d['ms_per_step'],1))
    else: print(l.strip())"; }
run "NAT_X=0"
run "NAT_FUSED_NTH=512 NAT_FUSED_SMEM_KB=120"
run "NAT_FUSED_SMEM_KB=120"
run "NAT_BENCH_WORKERS=4"
run "NAT_BENCH_WORKERS=8"
