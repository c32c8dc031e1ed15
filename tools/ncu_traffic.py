"""Per-launch DRAM traffic and duration of ncu --set full captures -> JSON
(profiles/<round>_ncu_traffic.json feeds bench.py's roofline "traffic").
Usage: python tools/ncu_traffic.py a.ncu-rep ... > traffic.json"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6,
         "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}

out = {}
for f in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    h, u, r = rows[0], rows[1], rows[2]

    def val(name):
        i = h.index(name)
        return float(r[i].replace(",", "")) * SCALE.get(u[i], 1.0)

    out[Path(f).stem] = {"kernel": r[h.index("Kernel Name")][:120],
                         "dram_read_bytes": val("dram__bytes_read.sum"),
                         "dram_write_bytes": val("dram__bytes_write.sum"),
                         "duration_s": val("gpu__time_duration.sum"),
                         "sm_clock_hz": val("sm__cycles_elapsed.avg.per_second") * 1e9
                         if u[h.index("sm__cycles_elapsed.avg.per_second")] == "Ghz" else None}
print(json.dumps(out, indent=1))
