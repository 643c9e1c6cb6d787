# A/B: packed far kernel compiled for 2 vs 3 resident CTAs per SM
for b in 3 2 3 2; do
  touch paper_2506_06190_b200/csrc/bem.cu
  NAT_NVCC_EXTRA="-DNAT_FAR_MINB=$b" python -m paper_2506_06190_b200.build > /dev/null || exit 1
  python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/b44_$b.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b44_$b.json'))
r=d['rooflines']; print('minb $b', round(d['value'],1), round(d['ms_per_step'],2), 'far_kernel', round(r['far_kernel']['frac'],3), round(r['far_kernel']['ms_per_step'],3), 'asm', round(d['phase_ms_per_step']['assembly'],3))"
done
