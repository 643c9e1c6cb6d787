python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 300 python scripts/mc_tail.py 0 2>&1 | tail -80
timeout 300 python scripts/mc_tail.py 63 2>&1 | tail -8
