"""One markdown row per kernel launch of an ncu --set full report (runs on the GPU box, so
only the small text summary travels back): duration, SM clock, DRAM read + write, MUFU (XU),
FMA and tensor pipe use, issue and warp activity, registers, the top three stall reasons
per issued instruction.  Usage: ncu_rows.py REPORT LABEL >> summary.md"""
import csv
import io
import re
import subprocess
import sys

rep, label = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
         "ns": 1e-9, "nsecond": 1e-9, "msecond": 1e-3, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6, "cycle/second": 1.0}


def g(d, name):
    i = col.get(name)
    if i is None:
        return float("nan")
    try:
        return float(d[i].replace(",", "")) * SCALE.get(units[i], 1.0)
    except ValueError:
        return float("nan")


for d in data:
    name = re.sub(r"\(.*", "", d[col["Kernel Name"]]).replace("void ", "").replace("<unnamed>::", "").replace("nat::", "")
    stalls = []
    for h, i in col.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
        if m:
            stalls.append((g(d, h), m.group(1)))
    stalls.sort(reverse=True)
    top = ", ".join(f"{n} {v:.2f}" for v, n in stalls[:3])
    dram = (g(d, "dram__bytes_read.sum") + g(d, "dram__bytes_write.sum")) / 1e6
    print(f"| {label} | {name.strip()} | {g(d, 'gpu__time_duration.sum') * 1e6:.1f} | "
          f"{g(d, 'sm__cycles_elapsed.avg.per_second') / 1e9:.3f} | {dram:.1f} | "
          f"{g(d, 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g(d, 'launch__registers_per_thread'):.0f} | {top} |")
