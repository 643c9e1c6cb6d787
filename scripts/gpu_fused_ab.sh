python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_mc.py tests/test_gpu_poisson.py -x -q > gpurun_out/pt_fused.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_fused.log
NAT_GMRES_FUSED=0 timeout 300 python scripts/prof_c4.py 0 2 2>&1 | tail -1
for kb in 120 0; do echo "smem cap $kb KB"; NAT_FUSED_SMEM_KB=$kb timeout 300 python scripts/prof_c4.py 0 2 2>&1 | tail -1; done
timeout 300 python scripts/prof_c4.py 0 1 > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:arnoldi_fused -s 100 -c 1 -o gpurun_out/fused_prof2 python scripts/prof_c4.py 0 1 > gpurun_out/ncu_fused.log 2>&1
echo "ncu rc=$?"
