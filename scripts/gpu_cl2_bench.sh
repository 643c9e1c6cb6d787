python -m paper_2506_06190_b200.build > /dev/null || exit 1
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for rep in 1 2; do for cl in 4 2; do echo "== bench CL $cl"; NAT_FUSED_CL=$cl timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1))"; done; done
echo "== bench CL 2 NTH 512"; NAT_FUSED_CL=2 NAT_FUSED_NTH=512 timeout 900 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1))"
