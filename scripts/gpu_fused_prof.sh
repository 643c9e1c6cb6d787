python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 300 python scripts/prof_c4.py 0 1 > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:arnoldi_fused -s 100 -c 1 -o gpurun_out/fused_prof python scripts/prof_c4.py 0 1 > gpurun_out/ncu_fused.log 2>&1
echo "ncu rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"arnoldi|givens|publish|dots|update|scale|radiate|stage|finish" --csv --log-file gpurun_out/fused_launches.csv python scripts/prof_c4.py 0 1 > /dev/null 2>&1; echo "list rc=$?"
