"""Host-side cost of one C2 step: cProfile of warm steps (GPU work is async,
so these are enqueue costs), plus host-enqueue vs GPU time per stage.

Usage: python tools/host_profile.py [--steps 3]
"""
import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2603_05353_b200 as P  # noqa: E402
from paper_2603_05353_b200 import pipeline as PL  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--chunk", type=int, default=2048)
    ap.add_argument("--ratio", type=float, default=0.15)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--reorder", action="store_true")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    cfg = bench.model_config(args)
    weights = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
    gen = P.generate_task(bench.make_task(args, cfg), seed=0)
    kvs = [P.prefill_chunk(weights, c) for c in gen.chunks]
    sel_cfg = P.SelectionConfig(ratio=args.ratio)

    def step():
        return P.assemble_select_recompute(weights, kvs, gen.chunks, gen.prompt_token_ids, sel_cfg)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    # host time of each stage call (no sync) vs the GPU's time for the step
    for _ in range(2):
        cache = P.assemble(kvs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        sel = P.run_selection(weights, gen.chunks, cache, gen.prompt_token_ids, sel_cfg)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"select: host enqueue {1e3 * (t1 - t0):.2f} ms, host until done {1e3 * (t2 - t0):.2f} ms, "
              f"gpu {e0.elapsed_time(e1):.2f} ms")
        plan = P.make_plan(cache, sel.selected)
        t0 = time.perf_counter()
        e0.record()
        P.recompute_selected(weights, cache, plan)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"recompute: host enqueue {1e3 * (t1 - t0):.2f} ms, host until done {1e3 * (t2 - t0):.2f} ms, "
              f"gpu {e0.elapsed_time(e1):.2f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(35)
    st.sort_stats("cumulative").print_stats(45)


if __name__ == "__main__":
    main()
