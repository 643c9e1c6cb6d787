python -m paper_2506_06190_b200.build > /dev/null || exit 1
NAT_DEBUG_PLAN=1 timeout 300 python scripts/mc_one.py 0 2>&1 | sort | uniq -c | head
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mc_finish_kernel --launch-skip 50 -c 1 -o gpurun_out/fin python scripts/mc_one.py 0 > gpurun_out/fin.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnoldi_fused --launch-skip 60 -c 1 -o gpurun_out/arn python scripts/mc_one.py 0 > gpurun_out/arn.log 2>&1; echo rc=$?
