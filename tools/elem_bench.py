"""A/B microbenchmark of the recompute-loop elementwise kernels at C2 shape
(4916 rows, d 4096): add_rmsnorm (no delta / fp32 delta) -> bf16.
Usage: python tools/elem_bench.py lib.so ..."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200 import _native as N  # noqa: E402


def timed(fn, iters=40):
    ts = []
    for i in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run(lib):
    N._lib = None
    N._fns.clear()
    N.load(Path(lib))
    from paper_2603_05353_b200 import engine as E

    S, d = 4916, 4096
    h = torch.randn(S, d, device="cuda")
    delta = torch.randn(S, d, device="cuda")
    g = torch.ones(d, device="cuda")
    t0 = timed(lambda: E.add_rmsnorm(h, None, 0, g, N.OUT_BF16))
    t1 = timed(lambda: E.add_rmsnorm(h, delta, 1, g, N.OUT_BF16))
    b0 = S * d * (4 + 2)
    b1 = S * d * (4 + 4 + 4 + 2)
    return [(t0, b0 / t0 / 1e6), (t1, b1 / t1 / 1e6)]


if __name__ == "__main__" and "--silu" not in sys.argv:
    for rep in range(2):
        for lib in sys.argv[1:]:
            r = run(lib)
            print(f"{lib}: rmsnorm {r[0][0] * 1e3:.1f} us {r[0][1]:.0f} GB/s | add+rmsnorm {r[1][0] * 1e3:.1f} us "
                  f"{r[1][1]:.0f} GB/s", flush=True)


def silu(lib):
    N._lib = None
    N._fns.clear()
    N.load(Path(lib))
    from paper_2603_05353_b200 import engine as E

    torch.manual_seed(0)
    S, dff = 4916, 14336
    gu = torch.randn(S, 2 * dff, device="cuda", dtype=torch.bfloat16)
    t = timed(lambda: E.silu_mul(gu, 1, dff, N.OUT_BF16))
    out = E.silu_mul(gu, 1, dff, N.OUT_BF16).float()
    g, u = gu[:, :dff].float(), gu[:, dff:].float()
    ref = torch.nn.functional.silu(g) * u
    err = float((out - ref).abs().max() / ref.abs().max())
    return t, S * dff * 6 / t / 1e6, err


if __name__ == "__main__" and "--silu" in sys.argv:
    for rep in range(2):
        for lib in [a for a in sys.argv[1:] if a != "--silu"]:
            t, gbs, err = silu(lib)
            print(f"{lib}: silu_mul {t * 1e3:.1f} us {gbs:.0f} GB/s rel err {err:.1e}", flush=True)
