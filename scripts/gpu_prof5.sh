python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 300 python scripts/prof_c4.py 0 1 > gpurun_out/plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"radiate_f32x2_kernel" -s 40 -c 1 -o gpurun_out/op_prof python scripts/prof_c4.py 0 1 > gpurun_out/ncu_op.log 2>&1; echo "ncu1 rc=$?"
