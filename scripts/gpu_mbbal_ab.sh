# Balanced wavenumber chunks (5-7) for the MC operator's tail launches: parity, per-n fractions, bench
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_multirank.py tests/test_gpu_configs.py -q -x 2>&1 | tail -1
for v in 0 1; do echo "== NAT_MB_BALANCE=$v"; NAT_MB_BALANCE=$v NAT_MC_GROUPS=1 timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "^ ?[0-9]+ |op total|without" | awk '{printf "%s | ", $0} END {print ""}' | cut -c1-2600; done
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for v in 0 1 0 1; do echo "== bench NAT_MB_BALANCE=$v"; NAT_MB_BALANCE=$v timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1), {k: round(v['frac'],3) for k,v in d['rooflines'].items()})"; done
