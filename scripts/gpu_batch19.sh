python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mc_launches.csv python scripts/mc_one.py 0 > gpurun_out/mc_one.log 2>&1; echo rc=$?
tail -3 gpurun_out/mc_one.log
