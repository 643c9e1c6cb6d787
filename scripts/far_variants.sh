# A/B of far-kernel shapes: rebuild with each (kTI, minBlocks) and time the bench phases
cp paper_2506_06190_b200/csrc/bem.cu /tmp/bem.cu.orig
for cfg in ${FAR_CFGS:-"16,3" "16,2" "16,3" "16,2"}; do
  ti=${cfg%,*}; mb=${cfg#*,}
  sed -i "s/^constexpr int kTI = [0-9]*;/constexpr int kTI = $ti;/; s/__launch_bounds__(kThreads, [0-9]) far_kernel_x2/__launch_bounds__(kThreads, $mb) far_kernel_x2/" paper_2506_06190_b200/csrc/bem.cu
  python -m paper_2506_06190_b200.build > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile-count --no-overlap > /tmp/b.json 2>/dev/null
  CFG=$cfg python - <<'P'
import json, os
d = json.load(open("/tmp/b.json"))
print(os.environ["CFG"], round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["phase_ms_per_step"].items()},
      d["clocks"]["sm_mhz"])
P
done
cp /tmp/bem.cu.orig paper_2506_06190_b200/csrc/bem.cu
