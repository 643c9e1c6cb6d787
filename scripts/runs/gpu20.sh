python -m paper_2506_06190_b200.build > /dev/null || exit 1
for ov in "" "--no-overlap"; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-profile-count $ov > gpurun_out/bench5$ov.json 2> gpurun_out/bench5$ov.err; echo "bench $ov rc=$?"
python - "gpurun_out/bench5$ov.json" <<'P'
import json,sys; d=json.load(open(sys.argv[1]))
print(d['value'], d['ms_per_step'], d['phase_ms_per_step'], d.get('phase_note'), d['e2e']['value'])
for k,v in d['rooflines'].items(): print(k, round(v['achieved'],1), round(v['frac'],3))
P
done
tail -3 gpurun_out/bench5.err
