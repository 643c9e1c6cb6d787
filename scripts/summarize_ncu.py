"""Summarise an ncu --set full report: per-kernel duration, DRAM traffic, pipe use.
Writes a markdown table to stdout and (optionally) profiles/traffic.json (bytes/launch)."""
import csv
import io
import json
import re
import subprocess
import sys

rep = sys.argv[1]
out_json = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def g(d, name, scale=1.0):
    i = col.get(name)
    try:
        return float(d[i]) * scale
    except (TypeError, ValueError):
        return float("nan")


def unit_scale(name):
    u = units[col[name]] if name in col else ""
    return {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
            "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}.get(u, 1.0)


print("| kernel | duration (us) | DRAM read (MB) | DRAM write (MB) | FMA pipe % | XU (MUFU) % | issue active % | warps active % | regs | SM clock (GHz) |")
print("|---|---|---|---|---|---|---|---|---|---|")
traffic = {}
for d in data:
    name = re.sub(r"\(.*", "", d[col["Kernel Name"]]).replace("void ", "").replace("<unnamed>::", "")
    dur = g(d, "gpu__time_duration.sum", unit_scale("gpu__time_duration.sum")) * 1e6
    rd = g(d, "dram__bytes_read.sum", unit_scale("dram__bytes_read.sum"))
    wr = g(d, "dram__bytes_write.sum", unit_scale("dram__bytes_write.sum"))
    print(f"| {name} | {dur:.1f} | {rd / 1e6:.2f} | {wr / 1e6:.2f} | "
          f"{g(d, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'launch__registers_per_thread'):.0f} | "
          f"{g(d, 'sm__cycles_elapsed.avg.per_second', unit_scale('sm__cycles_elapsed.avg.per_second')) / 1e9:.3f} |")
    base = name.split("<")[0]
    traffic.setdefault(base, rd + wr)
    traffic.setdefault(name.strip(), rd + wr)
if out_json:
    json.dump(traffic, open(out_json, "w"), indent=1)
