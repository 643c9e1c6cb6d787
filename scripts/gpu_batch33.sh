python -m paper_2506_06190_b200.build > /dev/null || exit 1
NAT_FUSED_NTH=256 timeout 600 python -m pytest tests/test_gpu_mc.py -q -x > gpurun_out/pt_b33.log 2>&1; echo "pytest nth256 rc=$?"; tail -1 gpurun_out/pt_b33.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
run() { echo "== $1"; env $1 timeout 600 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1))"; }
for rep in 1 2; do
run "NAT_X=0"
run "NAT_FUSED_NTH=256"
run "NAT_FUSED_NTH=256 NAT_FUSED_SMEM_KB=0"
run "NAT_FUSED_SMEM_KB=0"
done
echo "== serial call, nth 256"; NAT_FUSED_NTH=256 timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -1
