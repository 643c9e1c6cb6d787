# Givens steps on a side stream: parity and timing A/B (NAT_GIVENS_SIDE)
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_multirank.py tests/test_gpu_configs.py tests/test_gpu_bench_sweep.py tests/test_gpu_sweep.py -q -x 2>&1 | tail -1
for v in 0 1; do echo "== NAT_GIVENS_SIDE=$v"; NAT_GIVENS_SIDE=$v timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "iters|without" | cut -c1-150; NAT_GIVENS_SIDE=$v NAT_MC_GROUPS=2 timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "without" | sed 's/^/  G=2: /'; done
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for v in 0 1 0 1; do echo "== bench NAT_GIVENS_SIDE=$v"; NAT_GIVENS_SIDE=$v timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1), d['mc_gmres_iters']['mean'], d['mc_gmres_iters']['unconverged_systems'])"; done
