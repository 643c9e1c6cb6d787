python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnoldi_tma --launch-skip 100 -c 1 -o gpurun_out/tma python scripts/mc_one.py 0 > gpurun_out/tma.log 2>&1; echo rc=$?
timeout 600 env NAT_GMRES_TMA=0 ncu --set full --clock-control none --import-source on -k regex:arnoldi_fused_v2 --launch-skip 100 -c 1 -o gpurun_out/v2 python scripts/mc_one.py 0 > gpurun_out/v2.log 2>&1; echo rc=$?
