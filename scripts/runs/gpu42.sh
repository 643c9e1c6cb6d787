# fp64 sincos with constant-bank coefficients: fp64 parity + C5 measurements
python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_mf.py tests/test_gpu_bem.py tests/test_gpu_radiate.py tests/test_gpu_configs.py tests/test_gpu_galerkin.py tests/test_gpu_mc.py tests/test_gpu_bm.py -x -q > gpurun_out/pytest_42.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_42.log
timeout 900 python scripts/bench_configs.py C5_MF C5 > gpurun_out/configs_42.json 2> gpurun_out/configs_42.err; echo "cfg rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/configs_42.json'))
for k,v in d.items():
  if isinstance(v,dict): print(k, {a:b for a,b in v.items() if a!='note'})"
