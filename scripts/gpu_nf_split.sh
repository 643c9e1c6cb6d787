python -m paper_2506_06190_b200.build > /dev/null || exit 1
for r in 1024 512 2048 4096; do echo "== split rows $r"; NAT_NF_SPLIT_ROWS=$r timeout 300 python scripts/nf_time.py 2>&1 | tail -1; done
NAT_NF_SPLIT_ROWS=2048 timeout 300 python -m pytest tests/test_gpu_nf.py -q -x 2>&1 | tail -1
