python -m paper_2506_06190_b200.build > /dev/null || exit 1
for rep in 1 2; do NAT_BENCH_VERBOSE=1 timeout 1200 python bench.py > gpurun_out/bench_b36_$rep.json 2> gpurun_out/bench_b36_$rep.err; echo "bench rc=$?"; grep "step ms" gpurun_out/bench_b36_$rep.err; done
