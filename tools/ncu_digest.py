"""Digest of an ncu --set full report: headline metrics, stall reasons, sampled SASS regions."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
print(d.get("Kernel Name"))
for k in ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
          "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct", "smsp__warps_eligible.avg.per_cycle_active"]:
    if k in d:
        print(f"  {k} = {d[k]}")
st = []
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
print("  stalls/issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h, data = rows[1], rows[2:]
si, sc, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in data)
print(f"  samples {tot}, SASS lines {len(data)}")
# coarse regions: split at the hottest loop back-edge candidates = contiguous windows of 10 % of lines
n = len(data)
step = max(1, n // 12)
for a in range(0, n, step):
    s = sum(int(r[si] or 0) for r in data[a:a + step])
    e = sum(int(r[ie] or 0) for r in data[a:a + step])
    print(f"  [{a:5d},{a + step:5d}) samples {s:5d} ({100 * s / max(tot, 1):4.1f} %) inst {e}")
if len(sys.argv) > 2:
    top = sorted(range(n), key=lambda i: -int(data[i][si] or 0))[: int(sys.argv[2])]
    for i in sorted(top):
        print(f"  {i:5d} {data[i][si]:>5} {data[i][sc].strip()[:80]}")
