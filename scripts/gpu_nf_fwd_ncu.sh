python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nf_forward_fused -s 5 -c 1 -o /tmp/r02_nffwd python scripts/nf_time.py > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/ncu_rows.py /tmp/r02_nffwd.ncu-rep "NEXT-4 fused forward (5 products, 262,144 samples)" > gpurun_out/r02_nffwd_row.md
cat gpurun_out/r02_nffwd_row.md
