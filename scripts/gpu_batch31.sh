python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_nf.py -q -x > gpurun_out/pt_b31.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_b31.log
for L in 2 1 0; do echo "== smem levels $L"; NAT_NF_SMEM_LEVELS=$L timeout 300 python scripts/nf_time.py 2>&1 | tail -1; done
