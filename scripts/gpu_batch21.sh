python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_multirank.py tests/test_gpu_configs.py tests/test_gpu_sweep.py -q -x > gpurun_out/pt_b21.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_b21.log
echo "== default (finish v2, basis32)"; timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -5
echo "== NAT_BASIS32=0"; NAT_BASIS32=0 timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -5
echo "== NAT_BASIS32=0 NAT_GMRES_V2=1"; NAT_BASIS32=0 NAT_GMRES_V2=1 timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -5
