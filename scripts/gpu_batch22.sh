python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/mc_launches_warm.csv python scripts/mc_one.py 0 > gpurun_out/mc_one.log 2>&1; echo rc=$?
NAT_DEBUG_GMRES=1 timeout 300 python scripts/mc_one.py 0 2>&1 | tail -3
