"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
per-kernel table: launches, total ms, share of the captured step."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += ms
    total = sum(t for _, t in agg.values())
    print(f"| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| `{name[:80]}` | {n} | {t:.3f} | {100 * t / total:.1f}% |")
    print(f"| **total** | {sum(n for n, _ in agg.values())} | {total:.3f} | 100% |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
