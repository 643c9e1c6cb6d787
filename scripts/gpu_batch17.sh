python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python scripts/c2_orders.py 2>&1 | tail -12
