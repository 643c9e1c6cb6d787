# MC solve groups: parity, serial call time and the sweep bench for G = 1, 2, 4
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_mc.py -q -x -k "groups or surface_pressure or degenerate" 2>&1 | tail -1
for G in 1 2 4; do echo "== NAT_MC_GROUPS=$G"; NAT_MC_GROUPS=$G timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "op total|without"; NAT_MC_GROUPS=$G NAT_FUSED_NTH=256 NAT_FUSED_SMEM_KB=0 timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "without" | sed 's/^/  narrow: /'; done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for G in 1 2; do echo "== bench NAT_MC_GROUPS=$G"; NAT_MC_GROUPS=$G timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1), {k: round(v['frac'],3) for k,v in d['rooflines'].items()})"; done
