"""Correctness + timing of the tcgen05 pair GEMM (ifkv_gemm*) against torch /
cuBLAS on the recompute shapes (run on a B200: python tools/gemm_test.py)."""

import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_05353_b200 import _native as N  # noqa: E402
from paper_2603_05353_b200.build import build  # noqa: E402


def s():
    return torch.cuda.current_stream().cuda_stream


def rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30)).item()


def gemm(a, w, out_dtype=torch.bfloat16, acc=None, tile_n=0):
    M, K = a.shape
    Nn = w.shape[0]
    if acc is not None:
        out = acc
        N.call("ifkv_gemm", a.data_ptr(), a.stride(0), M, K, w.data_ptr(), Nn, N.IFKV_F32, out.data_ptr(), out.stride(0),
               1, tile_n, s())
        return out
    out = torch.empty((M, Nn), dtype=out_dtype, device=a.device)
    N.call("ifkv_gemm", a.data_ptr(), a.stride(0), M, K, w.data_ptr(), Nn,
           N.IFKV_F32 if out_dtype == torch.float32 else N.IFKV_BF16, out.data_ptr(), out.stride(0), 0, tile_n, s())
    return out


def check_plain():
    torch.manual_seed(0)
    for (M, K, Nn) in [(1, 64, 128), (5, 16, 96), (300, 512, 768), (257, 1024, 640), (4916, 4096, 2048), (700, 96, 200)]:
        for tn in (0, 1128, 1256, 1160, 1224):
            a = torch.randn(M, K, device="cuda").bfloat16()
            w = (torch.randn(Nn, K, device="cuda") / math.sqrt(K)).bfloat16()
            ref = a.float() @ w.float().t()
            o = gemm(a, w, tile_n=tn)
            o32 = gemm(a, w, torch.float32, tile_n=tn)
            h = torch.randn(M, Nn, device="cuda")
            h0 = h.clone()
            gemm(a, w, acc=h, tile_n=tn)
            torch.cuda.synchronize()
            e = (rel(o, ref), rel(o32, ref), rel(h - h0, ref))
            print(f"plain M={M} K={K} N={Nn} tn={tn}: bf16 {e[0]:.2e} f32 {e[1]:.2e} resid {e[2]:.2e}")
            assert e[0] < 1e-2 and e[1] < 1e-5 and e[2] < 1e-5, e


def check_qkv():
    torch.manual_seed(1)
    H, Hkv, Dh = 8, 2, 128
    for M in (37, 300, 1000):
        K = 512
        rows = 2048
        a = torch.randn(M, K, device="cuda").bfloat16()
        w = (torch.randn((H + 2 * Hkv) * Dh, K, device="cuda") / math.sqrt(K)).bfloat16()
        pos = torch.randint(0, 100000, (M,), device="cuda")
        cs = torch.empty((M, Dh // 2, 2), dtype=torch.float32, device="cuda")
        N.call("ifkv_rope_table", pos.data_ptr(), M, Dh, 500000.0, cs.data_ptr(), s())
        dst = torch.randperm(rows, device="cuda")[:M].contiguous()
        kd = torch.zeros(rows, Hkv, Dh, dtype=torch.bfloat16, device="cuda")
        vd = torch.zeros_like(kd)
        q = torch.empty(M, H, Dh, dtype=torch.bfloat16, device="cuda")
        N.call("ifkv_gemm_qkv_rope_scatter", a.data_ptr(), K, M, K, w.data_ptr(), H, Hkv, 0, cs.data_ptr(), q.data_ptr(),
               kd.data_ptr(), vd.data_ptr(), dst.data_ptr(), 1256 if M > 500 else 1128, s())
        ref = (a.float() @ w.float().t()).view(M, H + 2 * Hkv, Dh // 2, 2)
        c, sn = cs[:, None, :, 0], cs[:, None, :, 1]
        x, y = ref[..., 0], ref[..., 1]
        rot = torch.stack([x * c - y * sn, x * sn + y * c], -1).view(M, H + 2 * Hkv, Dh)
        torch.cuda.synchronize()
        e = (rel(q, rot[:, :H]), rel(kd[dst], rot[:, H:H + Hkv]), rel(vd[dst], ref.view(M, -1, Dh)[:, H + Hkv:]))
        untouched = torch.ones(rows, dtype=torch.bool, device="cuda")
        untouched[dst] = False
        z = kd[untouched].abs().max().item() if untouched.any() else 0.0
        print(f"qkv M={M}: q {e[0]:.2e} k {e[1]:.2e} v {e[2]:.2e} untouched {z}")
        assert max(e) < 1e-2 and z == 0
        # kv only
        kd2 = torch.zeros_like(kd)
        vd2 = torch.zeros_like(kd)
        N.call("ifkv_gemm_qkv_rope_scatter", a.data_ptr(), K, M, K, w[H * Dh:].contiguous().data_ptr(), H, Hkv, 1,
               cs.data_ptr(), None, kd2.data_ptr(), vd2.data_ptr(), dst.data_ptr(), 0, s())
        torch.cuda.synchronize()
        assert torch.equal(kd2, kd) and torch.equal(vd2, vd), "kv-only differs"


def check_swiglu():
    torch.manual_seed(2)
    for M, K, dff in [(300, 512, 1792), (4916, 1024, 512), (33, 64, 64)]:
        a = torch.randn(M, K, device="cuda").bfloat16()
        wg = (torch.randn(dff, K, device="cuda") / math.sqrt(K)).bfloat16()
        wu = (torch.randn(dff, K, device="cuda") / math.sqrt(K)).bfloat16()
        w = torch.stack([wg.view(dff // 64, 64, K), wu.view(dff // 64, 64, K)], 1).reshape(2 * dff, K).contiguous()
        out = torch.empty(M, dff, dtype=torch.bfloat16, device="cuda")
        for tn in (0, 1128, 1256):
            out.zero_()
            N.call("ifkv_gemm_swiglu", a.data_ptr(), K, M, K, w.data_ptr(), dff, out.data_ptr(), tn, s())
            g = a.float() @ wg.float().t()
            u = a.float() @ wu.float().t()
            e = rel(out, torch.nn.functional.silu(g) * u)
            assert e < 1e-2, (tn, e)
        g = a.float() @ wg.float().t()
        u = a.float() @ wu.float().t()
        ref = torch.nn.functional.silu(g) * u
        torch.cuda.synchronize()
        e = rel(out, ref)
        print(f"swiglu M={M} K={K} dff={dff}: {e:.2e}")
        assert e < 1e-2


def bench(fn, iters=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def timing():
    M = 4916
    shapes = [("qkv", 4096, 6144), ("o", 4096, 4096), ("gu", 4096, 28672), ("down", 14336, 4096), ("kv", 4096, 2048)]
    for name, K, Nn in shapes:
        a = torch.randn(M, K, device="cuda").bfloat16()
        w = (torch.randn(Nn, K, device="cuda") / math.sqrt(K)).bfloat16()
        wt = w.t().contiguous()  # round-1 layout [K, N] for cuBLAS
        fl = 2.0 * M * K * Nn
        t_cublas = bench(lambda: torch.mm(a, wt))
        res = {}
        for tn in (0, 1256, 1224, 1192, 1160):
            res[tn] = bench(lambda: gemm(a, w, tile_n=tn))
        line = " ".join(f"{tn or 'auto'}:{t*1e3:.0f}us({fl/t/1e9:.0f}TF)" for tn, t in res.items())
        print(f"{name:5s} M={M} K={K} N={Nn}: cublas {t_cublas*1e3:.0f}us ({fl/t_cublas/1e9:.0f} TF/s) | ours {line}")
    # fused epilogues at the C2 shapes
    K = 4096
    a = torch.randn(M, K, device="cuda").bfloat16()
    wgu = (torch.randn(28672, K, device="cuda") / 64).bfloat16()
    out = torch.empty(M, 14336, dtype=torch.bfloat16, device="cuda")
    for tn in (0, 1256, 1128):
        t = bench(lambda: N.call("ifkv_gemm_swiglu", a.data_ptr(), K, M, K, wgu.data_ptr(), 14336, out.data_ptr(), tn, s()))
        print(f"swiglu fused {tn}: {t*1e3:.0f}us ({2*M*K*28672/t/1e9:.0f} TF/s)")
    h = torch.randn(M, 4096, device="cuda")
    for name, K in (("o", 4096), ("down", 14336)):
        a = torch.randn(M, K, device="cuda").bfloat16()
        wo = (torch.randn(4096, K, device="cuda") / 64).bfloat16()
        wot = wo.t().contiguous()
        t = bench(lambda: torch.addmm(h, a, wot, out_dtype=torch.float32, out=h))
        print(f"residual {name} cublas addmm: {t*1e3:.0f}us ({2*M*K*4096/t/1e9:.0f} TF/s)")
        for tn in (0, 1256, 1192):
            t = bench(lambda: gemm(a, wo, acc=h, tile_n=tn))
            print(f"residual {name} {tn}: {t*1e3:.0f}us ({2*M*K*4096/t/1e9:.0f} TF/s)")


if __name__ == "__main__":
    build(verbose=True)
    N.load()
    check_plain()
    check_qkv()
    check_swiglu()
    if "--no-time" not in sys.argv:
        timing()
    print("gemm_test OK")
