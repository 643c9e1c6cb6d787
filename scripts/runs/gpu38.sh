# A/B: packed far kernel with 1 vs 2 interleaved column passes (NAT_FAR_UNROLL)
for u in 1 2 1 2; do
  touch paper_2506_06190_b200/csrc/bem.cu
  NAT_NVCC_EXTRA="-DNAT_FAR_UNROLL=$u" python -m paper_2506_06190_b200.build > /dev/null || exit 1
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/b38_$u.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b38_$u.json'))
r=d['rooflines']; print('unroll $u', round(d['value'],1), round(d['ms_per_step'],2), 'far_kernel', round(r['far_kernel']['frac'],3), r['far_kernel']['ms_per_step'], 'asm', round(d['phase_ms_per_step']['assembly'],3))"
done
