python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_mc.py tests/test_gpu_bem.py tests/test_gpu_multirank.py tests/test_gpu_mf.py -q -x > gpurun_out/pt_b8.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_b8.log
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_rep$r.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_rep$r.json'));print('rep',$r,round(d['value'],1),round(d['ms_per_step'],1),d['clocks'])"; done
timeout 300 python scripts/prof_c4.py 0 1 > gpurun_out/plain.log 2>&1 || exit 1
i=0
for spec in "radiate_f32x2_kernel<.int.2, .int.8, .int.2:0" "radiate_f32x2_kernel<.int.2, .int.8, .int.1:5" "radiate_f32x2_kernel<.int.2, .int.8, .int.0:0" "givens_kernel:100"; do
  k="${spec%%:*}"; sk="${spec##*:}"; i=$((i+1))
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s $sk -c 1 -o gpurun_out/r02_kk$i python scripts/prof_c4.py 0 1 > gpurun_out/r02_ncu_kk$i.log 2>&1; echo "ncu $k rc=$?"
done
