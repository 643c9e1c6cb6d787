python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1200 python scripts/sweep_shapes.py > gpurun_out/sweep_shapes.txt 2>&1; echo "rc=$?"; cat gpurun_out/sweep_shapes.txt | grep -v "^\[" | tail -40
