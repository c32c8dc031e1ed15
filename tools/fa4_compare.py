"""Diagnostic (not on the product path): how far is the recompute-attention
kernel (v5) from the public FlashAttention-4 CuTe-DSL forward kernel shipped
in the image (vllm.vllm_flash_attn.cute, a LIBRARY) on equal-FLOP shapes?

  * causal square, S tokens (ours: every token selected, horizon = its row)
  * C2 shape: 4916 queries at sorted random positions over 32768 keys (ours),
    vs FA4 non-causal 4916 x 16384 (the same FLOPs: mean horizon ~16K)

Timed interleaved with CUDA events.  python tools/fa4_compare.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_05353_b200 import engine as E  # noqa: E402

H, HKV, DH = 32, 8, 128


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    from vllm.vllm_flash_attn.cute.interface import flash_attn_func as fa4

    torch.manual_seed(0)
    rng = np.random.default_rng(0)
    cases = []
    for S in (8192, 16384):
        q = torch.randn(S, H, DH, device="cuda", dtype=torch.bfloat16)
        k = torch.randn(S, HKV, DH, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(S, HKV, DH, device="cuda", dtype=torch.bfloat16)
        hz = torch.arange(S, device="cuda", dtype=torch.int64)
        out = torch.empty_like(q)
        fl = 4.0 * H * DH * float(S) * (S + 1) / 2
        cases.append((f"causal S={S}", fl,
                      lambda q=q, k=k, v=v, hz=hz, out=out: E.recompute_attn(q, k, v, hz, H, HKV, DH, out=out),
                      lambda q=q, k=k, v=v: fa4(q[None], k[None], v[None], causal=True)))
    n, kq = 32768, 4916
    sel = np.sort(rng.choice(n, kq, replace=False))
    q = torch.randn(kq, H, DH, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(n, HKV, DH, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(n, HKV, DH, device="cuda", dtype=torch.bfloat16)
    hz = torch.as_tensor(sel, device="cuda")
    out = torch.empty_like(q)
    fl = 4.0 * H * DH * float(np.sum(sel + 1))
    sk = int(round(float(np.mean(sel + 1))))
    k2, v2 = k[:sk].contiguous(), v[:sk].contiguous()
    fl_fa = 4.0 * H * DH * kq * sk
    cases.append((f"C2 (ours sparse causal) / FA4 non-causal {kq}x{sk}", (fl, fl_fa),
                  lambda: E.recompute_attn(q, k, v, hz, H, HKV, DH, out=out),
                  lambda: fa4(q[None], k2[None], v2[None], causal=False)))
    for rep in range(3):
        for name, fl, ours, lib in cases:
            fo, ff = (fl, fl) if not isinstance(fl, tuple) else fl
            t_o = timeit(ours)
            try:
                t_f = timeit(lib)
                fa = f"FA4 {t_f:.3f} ms {ff / t_f / 1e9:.0f} TF/s"
            except Exception as e:  # noqa: BLE001
                fa = f"FA4 failed: {type(e).__name__}: {str(e)[:200]}"
            print(f"rep {rep} {name}: ours {t_o:.3f} ms {fo / t_o / 1e9:.0f} TF/s | {fa}", flush=True)


if __name__ == "__main__":
    main()
