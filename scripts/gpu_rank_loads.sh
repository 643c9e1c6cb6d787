# One rank's share of the C4 sweep at N = 8 / 4 / 2 (8 / 16 / 32 geometries) for several worker counts
python -m paper_2506_06190_b200.build > /dev/null || exit 1
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --no-profile-count"
for ng in 8 16 32; do for w in 6 8 12; do
  if [ $w -gt $ng ]; then continue; fi
  echo "== geometries $ng workers $w"; timeout 900 $B --geometries $ng --workers $w 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],1))"
done; done
