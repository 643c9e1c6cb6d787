python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_radiate.py tests/test_gpu_mc.py tests/test_gpu_configs.py -q -x > gpurun_out/pt_b5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_b5.log
timeout 300 python scripts/prof_c4.py 0 2 2>&1 | tail -1
timeout 600 python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline --no-e2e --no-profile-count > gpurun_out/bench_b5.json 2> gpurun_out/bench_b5.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_b5.json'));print(d['value'],d['ms_per_step']);[print(k,v['frac'],v['achieved']) for k,v in d['rooflines'].items()]"
