# Final: bench line (steps 5) + clocks, and ncu rows of the MC operator's tail launches
python -m paper_2506_06190_b200.build > /dev/null || exit 1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/r02_clocks.csv &
SMI=$!
NAT_BENCH_VERBOSE=1 timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
kill $SMI
rm -f gpurun_out/r02_tail_rows.md
for spec in "radiate_f32x2_kernel<.int.2, .int.4, .int.1:0" "radiate_f32x2_kernel<.int.2, .int.1, .int.1:0"; do
  k="${spec%%:*}"; sk="${spec##*:}"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s $sk -c 1 -o /tmp/r02_tail python scripts/prof_c4.py 0 1 > /dev/null 2>&1; echo "ncu $k rc=$?"
  python scripts/ncu_rows.py /tmp/r02_tail.ncu-rep "C4 MC operator tail launch" >> gpurun_out/r02_tail_rows.md
  rm -f /tmp/r02_tail.ncu-rep
done
