"""A/B microbenchmark of the fused rope + K/V scatter at the C2 recompute
shape (4916 rows x (32 + 2*8) heads x 128, bf16).  Usage: python tools/scatter_bench.py lib.so ..."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200 import _native as N  # noqa: E402


def run(lib, cold, iters=50):
    N._lib = None
    N._fns.clear()
    N.load(Path(lib))
    from paper_2603_05353_b200 import engine as E

    S, H, Hkv, Dh, n = 4916, 32, 8, 128, 32768
    rng = np.random.default_rng(0)
    sel = torch.as_tensor(np.sort(rng.choice(n, S, replace=False)), device="cuda")
    qkv = torch.randn(S, (H + 2 * Hkv) * Dh, device="cuda", dtype=torch.bfloat16)
    cs = E.rope_table(sel, Dh, 5e5, "cuda")
    q = torch.empty(S, H, Dh, device="cuda", dtype=torch.bfloat16)
    k = torch.zeros(n, Hkv, Dh, device="cuda", dtype=torch.bfloat16)
    v = torch.zeros_like(k)
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB, evicted by a READ (no dirty lines)
    ts = []
    for i in range(iters):
        if cold:
            flush.sum()
        else:
            qkv.add_(0)  # hot: the GEMM output just written, like inside the step
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        E.qkv_rope_scatter(qkv, 1, H, Hkv, Dh, cs, q, k, v, sel)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    byt = S * (H + 2 * Hkv) * Dh * 2 * 2
    return ms, byt / ms / 1e6


if __name__ == "__main__":
    for rep in range(2):
        for cold in (True, False):
            for lib in sys.argv[1:]:
                ms, gbs = run(lib, cold)
                print(f"{lib} {'cold' if cold else 'hot '}: {ms * 1e3:.1f} us  {gbs:.0f} GB/s", flush=True)
