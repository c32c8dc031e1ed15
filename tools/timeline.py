"""GPU timeline of one warm C2 step (torch.profiler / CUPTI, no nsys needed):
per-kernel totals, GPU idle gaps (time between kernels) and where they sit.

Usage: python tools/timeline.py [--ctx 32768] [--layers 0] [--out gpurun_out/timeline.json]
"""
import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2603_05353_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--chunk", type=int, default=2048)
    ap.add_argument("--ratio", type=float, default=0.15)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--reorder", action="store_true")
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    ap.add_argument("--steps", type=int, default=1, help="back-to-back steps inside the capture")
    ap.add_argument("--graph", action="store_true", help="replay the captured query graph (pipeline.QueryGraph)")
    args = ap.parse_args()
    cfg = bench.model_config(args)
    weights = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
    gen = P.generate_task(bench.make_task(args, cfg), seed=0)
    kvs = P.prefill_chunks(weights, gen.chunks)  # one store slab, as bench.py prepares the context
    sel_cfg = P.SelectionConfig(ratio=args.ratio)

    def step():
        return P.assemble_select_recompute(weights, kvs, gen.chunks, gen.prompt_token_ids, sel_cfg,
                                           reorder=args.reorder, graph=args.graph)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = []
    for e in evs:
        ks.append((e.time_range.start, e.time_range.end, e.name))
    ks.sort()
    t0, t1 = ks[0][0], max(k[1] for k in ks)
    busy = 0.0
    gaps = []
    cur_end = ks[0][0]
    prev = None
    for s, e, n in ks:
        if s > cur_end:
            gaps.append((s - cur_end, prev, n, cur_end - t0))
        busy += max(0, e - max(s, cur_end))
        cur_end = max(cur_end, e)
        prev = n
    tot = defaultdict(lambda: [0, 0.0])
    for s, e, n in ks:
        tot[n][0] += 1
        tot[n][1] += (e - s)
    span = (t1 - t0) / 1e3
    print(f"span {span:.3f} ms, busy {busy / 1e3:.3f} ms, idle {(t1 - t0 - busy) / 1e3:.3f} ms, {len(ks)} kernels")
    print("top kernels (ms total, launches):")
    for n, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
        print(f"  {d / 1e3:9.3f} {c:5d}  {n[:110]}")
    gaps.sort(key=lambda g: -g[0])
    print("largest gaps (us, at ms, after -> before):")
    for g, a, b, at in gaps[:25]:
        print(f"  {g:9.1f} @ {at / 1e3:8.3f}  {str(a)[:50]} -> {str(b)[:50]}")
    # the selection phase: from the first kernel to the first recompute GEMM
    first_gemm = next((s for s, e, n in ks if "gemm_pair" in n), t1)
    sel_k = [(s, e, n) for s, e, n in ks if s < first_gemm]
    sel_busy = defaultdict(float)
    for s, e, n in sel_k:
        sel_busy[n.split("(")[0][-60:]] += (e - s)
    sel_gap = sum(g for g, a, b, at in gaps if at + t0 < first_gemm)
    print(f"selection phase: {(first_gemm - t0) / 1e3:.3f} ms to the first recompute GEMM, "
          f"kernel time {sum(sel_busy.values()) / 1e3:.3f} ms, idle {sel_gap / 1e3:.3f} ms")
    for n, d in sorted(sel_busy.items(), key=lambda x: -x[1])[:16]:
        print(f"  {d / 1e3:8.3f}  {n}")
    # gap total per coarse phase (by position in the step)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"span_ms": span, "busy_ms": busy / 1e3,
                                          "kernels": [(s - t0, e - t0, n) for s, e, n in ks]}))


if __name__ == "__main__":
    main()
