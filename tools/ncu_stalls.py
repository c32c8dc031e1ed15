"""Top stalled SASS lines + pipe metrics of an ncu --set full capture.
Usage: python tools/ncu_stalls.py rep.ncu-rep [n]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, r = rows[0], rows[1], rows[2]
for i, name in enumerate(h):
    if re.search(r"gpu__time_duration.sum|sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"inst_executed_pipe_xu_realtime|sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active|"
                 r"pipe_alu_cycles_active.avg.pct_of_peak_sustained_active|pipe_fma_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"tc_wavefronts_mem_shared.sum.pct|lsu_wavefronts_mem_shared.sum.pct|smsp__inst_executed.sum$|"
                 r"sm__cycles_elapsed.avg.per_second|smsp__issue_active.avg.pct", name):
        print(f"{name:80s} {u[i]:6s} {r[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h, data = rows[1], rows[2:]
S, SS, IE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(x[SS] or 0) for x in data)
agg = {}
for x in data:
    for c in cols:
        agg[c] = agg.get(c, 0) + float(x[h.index(c)] or 0)
print("stall totals:", ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
for x in sorted(data, key=lambda x: -float(x[SS] or 0))[:n]:
    st = sorted(((float(x[h.index(c)] or 0), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{float(x[SS]) / tot * 100:5.1f}% {x[h.index('Address')][-5:]} {x[S][:64]:64s} {st[0][1]} {st[1][1]}")
