python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_nf.py -q -x > gpurun_out/pt_b29.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_b29.log
timeout 300 python scripts/nf_time.py 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/nf_launches.csv python scripts/nf_time.py > /dev/null 2>&1; echo ncu rc=$?
