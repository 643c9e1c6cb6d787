# row-sharded MC: parity tests + regression of the MC tests
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_mc.py tests/test_gpu_configs.py tests/test_gpu_timer.py -x -q > gpurun_out/pytest_45.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_45.log
python bench.py --steps 3 --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/b45.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b45.json')); print(d['value'], d['mc_gmres_iters'], round(d['rooflines']['mc_op_kernel']['frac'],3))"
