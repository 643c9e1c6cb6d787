# MC operator: resident CTAs per SM vs wave quantisation (NAT_RAD_OCC caps them via shared memory)
python -m paper_2506_06190_b200.build > /dev/null || exit 1
for o in 0 4 3; do echo "== NAT_RAD_OCC=$o"; NAT_RAD_OCC=$o NAT_DEBUG_PLAN=1 timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "kind 1 modes 64 |^64 |op total|without" | sort -u; done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for o in 0 4; do echo "== bench NAT_RAD_OCC=$o"; NAT_RAD_OCC=$o timeout 600 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1), {k: round(v['frac'],3) for k,v in d['rooflines'].items()})"; done
