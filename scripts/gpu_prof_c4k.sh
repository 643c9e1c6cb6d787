python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 300 python scripts/prof_c4.py 0 1 > gpurun_out/plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"radiate_f32x2_kernel|mc_finish" -s 40 -c 4 -o gpurun_out/c4k_prof python scripts/prof_c4.py 0 1 > gpurun_out/ncu_c4k.log 2>&1
echo "ncu rc=$?"
