# Pair kernel source-loop unroll (NAT_RAD_UNROLL) A/B: radiation and MC operator fractions
for u in 2 1 4 2; do
  touch paper_2506_06190_b200/csrc/radiate.cu
  NAT_NVCC_EXTRA="-DNAT_RAD_UNROLL=$u" python -m paper_2506_06190_b200.build > /dev/null || exit 1
  echo "== unroll $u"; timeout 300 python scripts/rad_frac.py 2>&1 | tail -2
done
