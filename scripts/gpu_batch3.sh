python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_radiate.py -q -x > gpurun_out/pt_b3.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_b3.log
timeout 600 python scripts/thin_wall_probe.py 2>&1 | tail -8
