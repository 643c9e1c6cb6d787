python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_radiate.py tests/test_gpu_configs.py tests/test_gpu_mc.py tests/test_gpu_sweep.py -q > gpurun_out/pt_b4.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_b4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_plain.log 2>&1; echo "smoke rc=$?"
timeout 1200 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/sanitizer_memcheck.log
