"""A/B microbenchmark of the recompute-attention kernel at the C2 shape:
4916 selected queries (uniform over 32768 positions) x 32 heads, 8 kv heads,
Dh 128, one layer.  Usage: python tools/attn_bench.py [lib.so ...]"""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_05353_b200 import _native as N  # noqa: E402


def run(lib, iters=30):
    torch.manual_seed(0)
    N._lib = None
    N.load(Path(lib))
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(0)
    n, k, Dh = int(os.environ.get("ATTN_N", "32768")), int(os.environ.get("ATTN_K", "4916")), 128
    H, Hkv = int(os.environ.get("ATTN_H", "32")), int(os.environ.get("ATTN_HKV", "8"))
    sel = np.sort(rng.choice(n, k, replace=False))
    q = torch.randn(k, H, Dh, device="cuda", dtype=torch.bfloat16)
    kk = torch.randn(n, Hkv, Dh, device="cuda", dtype=torch.bfloat16)
    vv = torch.randn(n, Hkv, Dh, device="cuda", dtype=torch.bfloat16)
    hz = torch.as_tensor(sel, device="cuda")
    out = torch.empty_like(q)
    for _ in range(3):
        E.recompute_attn(q, kk, vv, hz, H, Hkv, Dh, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        E.recompute_attn(q, kk, vv, hz, H, Hkv, Dh, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    flops = 4.0 * H * Dh * float(np.sum(sel + 1))
    return ms, flops / ms / 1e9, out.float()


if __name__ == "__main__":
    libs = sys.argv[1:] or [str(ROOT / "paper_2603_05353_b200/_build/libifkv.so")]
    ref = None
    for rep in range(4):
        for lib in libs:
            ms, tf, out = run(lib)
            if ref is None:
                ref = out
            err = float((out - ref).abs().max() / ref.abs().max())
            print(f"{lib}: {ms:.3f} ms  {tf:.0f} TFLOP/s  (max rel diff vs first lib {err:.1e})", flush=True)
