"""Rebuild profiles/ncu_summary.json from ncu --set full reports (one kernel launch each).

  python tools/ncu_summary.py key=report.ncu-rep:nodes:"what" ...
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_summary.json")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (val, u) for k, u, val in zip(h, units, v)}


def num(d, k, scale_units=True):
    if k not in d:
        return None
    val, unit = d[k]
    try:
        x = float(val.replace(",", ""))
    except ValueError:
        return None
    if scale_units:
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "usecond": 1, "us": 1,
              "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1)
    return x


summary = json.load(open(OUT)) if os.path.exists(OUT) else {}
for arg in sys.argv[1:]:
    key, rest = arg.split("=", 1)
    rep, nodes, what = rest.split(":", 2)
    d = raw(rep)
    rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
    inst = num(d, "smsp__inst_executed.sum", False)
    summary[key] = {
        "what": what,
        "kernel": d.get("Kernel Name", ("", ""))[0],
        "report": os.path.basename(rep),
        "duration_us": num(d, "gpu__time_duration.sum"),
        "dram_read": rd, "dram_write": wr,
        "dram_bytes_per_launch": (rd or 0) + (wr or 0),
        "fp64_pipe_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", False),
        "fma_pipe_pct": num(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", False),
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active", False),
        "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active", False),
        "regs": num(d, "launch__registers_per_thread", False),
        "grid": num(d, "launch__grid_size", False),
        "inst_per_node": (inst * 32.0 / float(nodes)) if inst else None,
    }
    print(key, json.dumps(summary[key]))
json.dump(summary, open(OUT, "w"), indent=1)
