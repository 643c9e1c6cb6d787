python -m paper_2506_06190_b200.build > /dev/null || exit 1
for W in 1 2 4; do
  timeout 600 python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count --workers $W > gpurun_out/bench_w$W.json 2> gpurun_out/bench_w$W.err
  echo "W=$W rc=$?"
done
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "full rc=$?"
