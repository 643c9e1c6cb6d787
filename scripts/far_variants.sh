# A/B of far-kernel tile shapes: rebuild with each (kTI, minBlocks) and time the bench phases
for cfg in "16 3" "8 3" "8 4" "32 2"; do
  set -- $cfg
  sed -i "s/^constexpr int kTI = [0-9]*;/constexpr int kTI = $1;/; s/__launch_bounds__(kThreads, [0-9]) far_kernel_x2/__launch_bounds__(kThreads, $2) far_kernel_x2/" paper_2506_06190_b200/csrc/bem.cu
  python -m paper_2506_06190_b200.build > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile-count 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('kTI=$1 minB=$2', d['ms_per_step'], d['phase_ms_per_step']['assembly'])"
done
