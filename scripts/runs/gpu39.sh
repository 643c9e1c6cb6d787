# MC split-K reduced in thread-block clusters (DSMEM): parity + A/B (NAT_MC_NOCLUSTER)
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1200 python -m pytest tests/test_gpu_mc.py tests/test_gpu_configs.py tests/test_gpu_poisson.py -x -q > gpurun_out/pytest_39.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_39.log
for mode in cluster nocluster cluster nocluster; do
  if [ $mode = nocluster ]; then export NAT_MC_NOCLUSTER=1; else unset NAT_MC_NOCLUSTER; fi
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/b39_$mode.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b39_$mode.json'))
r=d['rooflines']; print('$mode', round(d['value'],1), round(d['ms_per_step'],2), 'mc_op_kernel', round(r['mc_op_kernel']['frac'],3), 'mc_operator', round(r['mc_operator']['frac'],3), 'mc_solve ms', round(d['phase_ms_per_step']['mc_solve'],2), 'iters', d['mc_gmres_iters'])"
done
