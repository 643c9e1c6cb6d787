python -m paper_2506_06190_b200.build > /dev/null || exit 1
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for p in 1 0 1 0; do echo "== NAT_BENCH_PRIO=$p"; NAT_BENCH_PRIO=$p timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1))"; done
