# arithmetic-progression recurrence in the multi-wavenumber kernels: parity + C3/C4 A/B
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_radiate.py tests/test_gpu_mc.py -x -q > gpurun_out/pytest_43.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_43.log
for mode in arith direct; do
  if [ $mode = direct ]; then export NAT_NO_ARITH=1; else unset NAT_NO_ARITH; fi
  timeout 900 python scripts/bench_configs.py C3 C4 > gpurun_out/configs_43_$mode.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/configs_43_$mode.json'))
c3=d['C3']; c4=d['C4']
print('$mode', 'C3 mc', round(c3['mc_solve_seconds']*1e3,2), 'ms rad', round(c3['radiation_seconds']*1e3,3), 'ms', round(c3['radiation_pair_modes_per_s']/1e12,3), 'T | C4 mc', round(c4['mc_solve_seconds']*1e3,2), 'ms rad', round(c4['radiation_seconds']*1e3,2), 'ms', round(c4['radiation_pair_modes_per_s']/1e12,3), 'T', c3.get('mc_iters')[:4])"
done
