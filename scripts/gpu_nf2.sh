python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_nf.py tests/test_gpu_timer.py -q -x > gpurun_out/pt_nf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_nf.log
timeout 600 python -c "
import sys, json, torch; sys.path.insert(0,'.')
import bench_secondary as S
from paper_2506_06190_b200 import nat
torch.cuda.set_device(0)
print(json.dumps(S.run_nf(nat, torch, 10, peaks=json.load(open('MEASURED_PEAKS.json')))))
" > gpurun_out/nf_bench.json 2>&1; cat gpurun_out/nf_bench.json | tail -2
cat > /tmp/nfprof.py <<'PY'
import sys, json, torch; sys.path.insert(0,'.')
import bench_secondary as S
from paper_2506_06190_b200 import nat
torch.cuda.set_device(0)
S.run_nf(nat, torch, 2)
PY
timeout 300 python /tmp/nfprof.py > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nf_launches.csv python /tmp/nfprof.py > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nf_gemm -s 30 -c 2 -o gpurun_out/nf_gemm_prof python /tmp/nfprof.py > /dev/null 2>&1; echo "ncu rc=$?"
