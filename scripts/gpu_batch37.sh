python -m paper_2506_06190_b200.build > /dev/null || exit 1
nproc; NAT_BENCH_VERBOSE=1 timeout 1200 python bench.py --steps 6 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/bench_b37.json 2> gpurun_out/bench_b37.err; echo "bench rc=$?"; grep "\[bench\]" gpurun_out/bench_b37.err
