python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_multirank.py tests/test_gpu_configs.py tests/test_gpu_sweep.py tests/test_gpu_bem.py -q -x > gpurun_out/pt_b23.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_b23.log
echo "== default (tma, basis32)"; timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -3
echo "== tma fp64 basis"; NAT_BASIS32=0 timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -3
echo "== v2 fp32"; NAT_GMRES_TMA=0 timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/mc_launches_tma.csv python scripts/mc_one.py 0 > gpurun_out/mc_one.log 2>&1; echo rc=$?
