# Narrower wavenumber chunks for the MC operators' underfilled tail launches: per-n fractions, parity, bench A/B
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_mc.py tests/test_gpu_multirank.py -q -x 2>&1 | tail -1
for v in 1 0; do echo "== NAT_MB_FIXED=$v"; if [ $v = 1 ]; then export NAT_MB_FIXED=1; else unset NAT_MB_FIXED; fi; timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "^ ?[0-9]+ |op total|without" | awk '{printf "%s | ", $0} END {print ""}'; done
unset NAT_MB_FIXED
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for v in 1 0 1 0; do echo "== bench NAT_MB_FIXED=$v"; if [ $v = 1 ]; then export NAT_MB_FIXED=1; else unset NAT_MB_FIXED; fi; timeout 600 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1), round(d['rooflines']['mc_operator_kernel']['frac'],3))"; done
