# A/B of the MC split rule on the same box: overlapped step value and per-kernel rooflines
python -m paper_2506_06190_b200.build > /dev/null || exit 1
for rep in 1 2; do
for mode in coarse fine coarse fine; do
  if [ $mode = coarse ]; then export NAT_MC_COARSE=1; else unset NAT_MC_COARSE; fi
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/ab_$mode.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$mode.json'))
r=d['rooflines']; print('$mode', round(d['value'],1), round(d['ms_per_step'],2), 'mc_op_kernel', round(r['mc_op_kernel']['frac'],3), 'mc_operator', round(r['mc_operator']['frac'],3), 'mc_solve ms', round(d['phase_ms_per_step']['mc_solve'],2))"
done
done
