python -m paper_2506_06190_b200.build > /dev/null || exit 1
NAT_RAD_NPOLY=2 timeout 600 python -m pytest tests/test_gpu_radiate.py tests/test_gpu_mc.py -q -x > gpurun_out/pt_b32.log 2>&1; echo "pytest npoly2 rc=$?"; tail -2 gpurun_out/pt_b32.log
for np in 0 1 2 3; do echo "== npoly $np"; NAT_RAD_NPOLY=$np timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "^64 |op total|without"; NAT_RAD_NPOLY=$np timeout 300 python scripts/prof_c4.py 0 2 2>&1 | tail -1; done
