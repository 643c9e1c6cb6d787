python -m paper_2506_06190_b200.build > /dev/null || exit 1
python scripts/prof_mc.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"radiate_f32x2" -s 2 -c 2 \
    -o gpurun_out/prof_mc2 python scripts/prof_mc.py > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
