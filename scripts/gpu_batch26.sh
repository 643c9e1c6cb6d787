python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_mc.py tests/test_gpu_multirank.py tests/test_gpu_configs.py tests/test_gpu_sweep.py tests/test_gpu_bem.py -q -x > gpurun_out/pt_b26.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_b26.log
echo "== default"; timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -2
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
for v in 1 0 1 0; do echo "== bench NAT_BASIS32=$v"; NAT_BASIS32=$v timeout 600 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mc_finish --launch-skip 50 -c 1 -o gpurun_out/fin2 python scripts/mc_one.py 0 > gpurun_out/fin2.log 2>&1; echo rc=$?
