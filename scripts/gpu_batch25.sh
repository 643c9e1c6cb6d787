python -m paper_2506_06190_b200.build > /dev/null || exit 1
NAT_DEBUG_PLAN=1 timeout 300 python scripts/mc_one.py 0 2>&1 | grep "kind 1 modes 64 " | head -2
for pl in "" "2,128,2,8,1" "2,128,4,8,1" "2,256,1,8,1" "2,256,2,8,1" "4,128,1,8,1" "4,128,2,8,1"; do
  echo "== plan [$pl]"; NAT_RAD_PLAN=$pl timeout 300 python scripts/mc_tail.py 0 2>&1 | grep -E "^64 |op total|without"
done
