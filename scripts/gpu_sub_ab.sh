# MC operator tail: 2-4 CTAs per source tile when the grid leaves SMs idle (NAT_RAD_SUB A/B)
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_radiate.py tests/test_gpu_multirank.py -q -x 2>&1 | tail -1
for v in 0 1; do echo "== NAT_RAD_SUB=$v"; NAT_RAD_SUB=$v NAT_MC_GROUPS=1 timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "^ ?[0-9]+ |op total|without" | awk '{printf "%s | ", $0} END {print ""}' | cut -c1-900; NAT_RAD_SUB=$v timeout 300 python scripts/prof_c4.py 0 2 2>&1 | tail -1; done
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for v in 0 1 0 1; do echo "== bench NAT_RAD_SUB=$v"; NAT_RAD_SUB=$v timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1), {k: round(v['frac'],3) for k,v in d['rooflines'].items()}, round(d['mc_call']['frac'],3))"; done
