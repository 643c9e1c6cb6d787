python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python scripts/c3_groups.py 2>&1 | tail -5
echo "== CL 2, NTH 256"; NAT_FUSED_CL=2 NAT_FUSED_NTH=256 NAT_FUSED_SMEM_KB=0 timeout 600 python scripts/c3_groups.py 2>&1 | tail -5
