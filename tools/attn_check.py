"""Recompute attention (tcgen05) A/B: correctness against a torch fp32
reference (small cases: ragged tiles, G = 4 / 7, key splits, key ranges) and
v5 at the C2 shape, then interleaved timing of several library variants.
Usage: python tools/attn_check.py [name=lib.so:gen ...]  (gen: IFKV_ATTN_GEN of the library, 5 today)"""
import math
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200 import _native as N  # noqa: E402


def use(lib, gen):
    N._lib = None
    N._fns.clear() if hasattr(N, "_fns") else None
    N.load(Path(lib))
    os.environ["IFKV_ATTN_GEN"] = str(gen)
    from paper_2603_05353_b200 import engine as E

    return E


def ref_attn(q, k, v, hz, H, Hkv, ks=None):
    S, _, Dh = q.shape
    G = H // Hkv
    out = torch.empty(S, H, Dh, dtype=torch.float32, device=q.device)
    kf, vf = k.float(), v.float()
    for t in range(S):
        lo = 0 if ks is None else int(ks[t])
        hi = int(hz[t]) + 1
        for g in range(Hkv):
            qq = q[t, g * G:(g + 1) * G].float()
            s = qq @ kf[lo:hi, g].T / math.sqrt(Dh)
            p = torch.softmax(s, -1)
            out[t, g * G:(g + 1) * G] = p @ vf[lo:hi, g]
    return out


def case(E, n, k, H, Hkv, seed, ranged=False):
    g = torch.Generator(device="cpu").manual_seed(seed)
    rng = np.random.default_rng(seed)
    sel = np.sort(rng.choice(n, k, replace=False))
    q = torch.randn(k, H, 128, generator=g).to("cuda", torch.bfloat16)
    kk = torch.randn(n, Hkv, 128, generator=g).to("cuda", torch.bfloat16)
    vv = torch.randn(n, Hkv, 128, generator=g).to("cuda", torch.bfloat16)
    hz = torch.as_tensor(sel, device="cuda")
    ks = None
    if ranged:
        ks = torch.as_tensor(np.maximum(sel - rng.integers(0, 700, k), 0), device="cuda")
    out = E.recompute_attn(q, kk, vv, hz, H, Hkv, 128, key_start=ks)
    torch.cuda.synchronize()
    return q, kk, vv, hz, ks, out


def check_small(E, tag):
    worst = 0.0
    for (n, k, H, Hkv, ranged) in [(700, 37, 8, 2, False), (1500, 300, 32, 8, False), (2048, 130, 28, 4, False),
                                   (4096, 520, 32, 8, True), (3000, 1000, 32, 8, False), (513, 513, 4, 1, False)]:
        q, kk, vv, hz, ks, out = case(E, n, k, H, Hkv, n + k)
        if ranged:
            q, kk, vv, hz, ks, out = case(E, n, k, H, Hkv, n + k, ranged=True)
        r = ref_attn(q, kk, vv, hz.cpu(), H, Hkv, None if ks is None else ks.cpu())
        err = float((out.float() - r).abs().max() / r.abs().max())
        worst = max(worst, err)
        print(f"{tag} n={n} k={k} H={H} Hkv={Hkv} ranged={ranged}: max rel err vs fp32 torch {err:.2e}", flush=True)
    return worst


def time_c2(E, iters=20, k=4916, n=32768, H=32, Hkv=8):
    rng = np.random.default_rng(0)
    sel = np.sort(rng.choice(n, k, replace=False))
    torch.manual_seed(0)
    q = torch.randn(k, H, 128, device="cuda", dtype=torch.bfloat16)
    kk = torch.randn(n, Hkv, 128, device="cuda", dtype=torch.bfloat16)
    vv = torch.randn(n, Hkv, 128, device="cuda", dtype=torch.bfloat16)
    hz = torch.as_tensor(sel, device="cuda")
    out = torch.empty_like(q)
    for _ in range(3):
        E.recompute_attn(q, kk, vv, hz, H, Hkv, 128, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        E.recompute_attn(q, kk, vv, hz, H, Hkv, 128, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    return ms, 4.0 * H * 128 * float(np.sum(sel + 1)) / ms / 1e9, out.float()


if __name__ == "__main__":
    base = str(ROOT / "paper_2603_05353_b200/_build/libifkv.so")
    specs = sys.argv[1:] or [f"v5={base}:5", f"v7={base}:7"]
    variants = []
    for s in specs:
        name, _, rest = s.partition("=")
        lib, _, gen = rest.rpartition(":")
        variants.append((name, lib, int(gen)))
    for name, lib, gen in variants:
        E = use(lib, gen)
        check_small(E, name)
    ref = None
    for shape in [dict(), dict(H=28, Hkv=4, k=4916), dict(k=1639)]:
        for rep in range(3):
            for name, lib, gen in variants:
                E = use(lib, gen)
                ms, tf, out = time_c2(E, **shape)
                if rep == 0 and name == variants[0][0]:
                    ref = out
                err = float((out - ref).abs().max() / ref.abs().max())
                print(f"{shape or 'C2'} {name}: {ms:.3f} ms {tf:.0f} TFLOP/s (max rel diff vs {variants[0][0]} {err:.1e})",
                      flush=True)
