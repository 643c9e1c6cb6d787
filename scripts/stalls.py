"""Top warp-stall reasons per kernel of an ncu --set full report (cycles per issued
instruction, smsp__average_warps_issue_stalled_*_per_issue_active)."""
import csv
import io
import re
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
pat = re.compile(r"smsp__average_warps_issue_stalled_(.+)_per_issue_active\.ratio")
cols = [(i, pat.match(h).group(1)) for i, h in enumerate(hdr) if pat.match(h)]
ki = hdr.index("Kernel Name")
for d in data:
    name = re.sub(r"\(.*", "", d[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
    vals = []
    for i, nm in cols:
        try:
            vals.append((float(d[i]), nm))
        except ValueError:
            pass
    vals.sort(reverse=True)
    print(f"{name[:60]:60s} " + ", ".join(f"{nm} {v:.2f}" for v, nm in vals[:7]))
