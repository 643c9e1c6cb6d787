# A/B of the dense-chain order in the overlapped bench step
python -m paper_2506_06190_b200.build > /dev/null || exit 1
for rep in 1 2; do
for order in asm_first interleave; do
  NAT_BENCH_ORDER=$order python bench.py --steps 5 --no-cpu-baseline --no-profile-count > gpurun_out/b40_$order.json 2>gpurun_out/b40_$order.err
  python -c "
import json; d=json.load(open('gpurun_out/b40_$order.json'))
print('$order', round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), {k:round(v,2) for k,v in d['phase_ms_per_step'].items()}, d['gmres_iters'], d['mc_gmres_iters'])" || tail -3 gpurun_out/b40_$order.err
done
done
