python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_nf.py -q -x > gpurun_out/pt_nf.log 2>&1; echo "pytest rc=$?"; tail -40 gpurun_out/pt_nf.log
