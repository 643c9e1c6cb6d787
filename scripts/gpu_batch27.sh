python -m paper_2506_06190_b200.build > /dev/null || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:mc_finish --csv --log-file gpurun_out/fin_launches.csv python scripts/mc_one.py 0 > /dev/null 2>&1; echo rc=$?
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/fin_launches.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
v=[float(r[vi].replace(',','')) for r in rows[1:]]
print('finish launches', len(v), 'total ms', sum(v)/1e6, 'median us', sorted(v)[len(v)//2]/1e3)
PY
