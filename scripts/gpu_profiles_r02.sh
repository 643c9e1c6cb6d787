# Round-2 evidence: full bench line (C4 headline + secondary), clocks during it, launch list
# of the bench command (2 geometries, 1 worker), ncu --set full of the main kernels of one C4
# geometry (prof_c4.py), of the neural field's tensor-core products and of the C2 multi-
# wavenumber far kernel; everything under gpurun_out/r02_*.
python -m paper_2506_06190_b200.build > /dev/null || exit 1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/r02_clocks.csv &
SMI=$!
NAT_BENCH_VERBOSE=1 timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
kill $SMI
CMD="python bench.py --steps 1 --warmup 1 --geometries 2 --workers 1 --no-secondary --no-e2e --no-cpu-baseline --no-profile-count"
timeout 600 $CMD > gpurun_out/r02_launch_plain.json 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_launch_ncu.log 2>&1; echo "launches rc=$?"
timeout 300 python scripts/prof_c4.py 0 1 > gpurun_out/plain.log 2>&1 || exit 1
i=0
for spec in "radiate_f32x2_kernel<.int.2, .int.8, .int.2:0" "radiate_f32x2_kernel<.int.2, .int.8, .int.1:5" "radiate_f32x2_kernel<.int.2, .int.8, .int.0:0" "arnoldi_fused_v2:100" "mc_finish:5" "stage_kernel:5" "givens_kernel:100"; do
  k="${spec%%:*}"; sk="${spec##*:}"; i=$((i+1))
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s $sk -c 1 -o /tmp/r02_k$i python scripts/prof_c4.py 0 1 > /tmp/r02_ncu_k$i.log 2>&1; echo "ncu $k rc=$?"
  python scripts/ncu_rows.py /tmp/r02_k$i.ncu-rep "C4 $k" >> gpurun_out/r02_ncu_rows.md
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nf_gemm -s 20 -c 4 -o /tmp/r02_nf python scripts/nf_time.py > /dev/null 2>&1; echo "ncu nf rc=$?"
python scripts/ncu_rows.py /tmp/r02_nf.ncu-rep "NEXT-4 layer products" >> gpurun_out/r02_ncu_rows.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:far_kernel_multi -s 1 -c 1 -o /tmp/r02_far python scripts/c2_far_multi.py > /dev/null 2>&1; echo "ncu far rc=$?"
python scripts/ncu_rows.py /tmp/r02_far.ncu-rep "C2 far (3 wavenumbers)" >> gpurun_out/r02_ncu_rows.md
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r02_nf_launches.csv python scripts/nf_time.py > /dev/null 2>&1; echo "nf launches rc=$?"
du -sh gpurun_out
