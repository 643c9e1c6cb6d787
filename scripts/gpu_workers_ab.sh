python -m paper_2506_06190_b200.build > /dev/null || exit 1
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for w in 6 8 10 6 8; do echo "== workers $w"; timeout 900 $B --workers $w 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1))"; done
