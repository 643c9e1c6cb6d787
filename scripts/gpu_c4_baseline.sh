python -m paper_2506_06190_b200.build > /dev/null || exit 1
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
NAT_DEBUG_GMRES=1 timeout 300 python scripts/prof_c4.py 0 3 > gpurun_out/c4_0.log 2>&1
NAT_DEBUG_GMRES=1 timeout 300 python scripts/prof_c4.py 63 2 > gpurun_out/c4_63.log 2>&1
timeout 600 python scripts/bench_configs.py C4_SWEEP > gpurun_out/c4_sweep.json 2> gpurun_out/c4_sweep.err
timeout 600 python scripts/prof_c4.py 0 1 > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/prof_c4.py 0 1 > gpurun_out/ncu.log 2>&1
echo done
