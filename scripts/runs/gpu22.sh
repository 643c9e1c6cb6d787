# Sanity pass of the restored tree: GPU tests, smoke, default bench line.
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r22.json 2> gpurun_out/bench_r22.err; echo "bench rc=$?"
cat gpurun_out/bench_r22.json | head -c 600
