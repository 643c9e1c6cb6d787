# NEXT-4: parity tests and the training-step timing
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_nf.py -q -x 2>&1 | tail -1
timeout 300 python scripts/nf_time.py 2>&1 | tail -2
echo "== unfused forward (A/B)"; NAT_NF_FUSED=0 timeout 300 python scripts/nf_time.py 2>&1 | tail -1
