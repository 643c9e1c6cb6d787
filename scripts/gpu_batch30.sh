python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nf_gemm_persist --launch-skip 11 -c 1 -o gpurun_out/nfg python scripts/nf_time.py > gpurun_out/nfg.log 2>&1; echo rc=$?
