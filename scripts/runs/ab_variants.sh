# A/B the prebuilt libnat variants (scripts/build_variants.sh) on the bench phases; the
# in-tree libnat.so is restored afterwards.  Usage: bash scripts/runs/ab_variants.sh base cc16 ...
P=paper_2506_06190_b200
cp $P/libnat.so /tmp/libnat_base.so
for round in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/libnat_base.so $P/libnat.so; else cp $P/_variants/libnat_$v.so $P/libnat.so; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-profile-count --no-overlap > /tmp/b.json 2>/tmp/b.err || { echo "$v failed"; tail -3 /tmp/b.err; continue; }
  V=$v python - <<'P'
import json, os
d = json.load(open("/tmp/b.json"))
r = d["rooflines"]
print(os.environ["V"], round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["phase_ms_per_step"].items()},
      "far frac", round(r["far_kernel"]["frac"], 4), "far ms", round(r["far_kernel"]["ms_per_step"], 3), d["clocks"]["sm_mhz"])
P
done
done
cp /tmp/libnat_base.so $P/libnat.so
