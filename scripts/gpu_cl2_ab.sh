# Fused Arnoldi with 2 CTAs per system (one wave of 128 CTAs for 64 systems) vs 4
python -m paper_2506_06190_b200.build > /dev/null || exit 1
NAT_FUSED_CL=2 timeout 600 python -m pytest tests/test_gpu_mc.py -q -x -k "surface_pressure or groups or c3_launch" 2>&1 | tail -1
for cl in 4 2; do echo "== CL $cl"; NAT_FUSED_CL=$cl timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "without"; NAT_FUSED_CL=$cl NAT_MC_GROUPS=2 timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "without" | sed 's/^/  G=2: /'; done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for cl in 4 2; do echo "== bench CL $cl"; NAT_FUSED_CL=$cl timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1))"; done
