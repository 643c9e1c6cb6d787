python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
