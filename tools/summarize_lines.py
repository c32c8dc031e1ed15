"""Markdown table of bench JSON lines (last line of each log)."""
import json
import sys
from pathlib import Path

print("| run | workload | ms/step | ctx tok/s | stages ms (asm / select / recompute) | full prefill ms | ratio | attn TF/s (frac) |")
print("|---|---|---:|---:|---|---:|---:|---|")
for f in sys.argv[1:]:
    lines = [l for l in Path(f).read_text().splitlines() if l.startswith("{")]
    if not lines:
        continue
    d = json.loads(lines[-1])
    st = d.get("stages_ms", {})
    stages = " / ".join(f"{v:.1f}" for v in st.values())
    r = d.get("roofline") or {}
    ach = r.get("achieved")
    print(f"| {Path(f).stem} | {d['config']['workload']} | {d['ms_per_step']:.1f} | {d['value']:.0f} | {stages} | "
          f"{d.get('full_prefill_ms', 0):.0f} | {d.get('ratio_vs_full_prefill', 0):.3f} | "
          f"{ach:.0f} ({r.get('frac', 0):.2f}) |" if ach else "| |")
