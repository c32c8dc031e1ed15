"""ifkv_prompt_mm vs cuBLAS for the scoring-pass GEMM shapes (C2: 3 split
terms x 32 prompt rows), weights cycled over copies larger than L2.
Usage: python tools/prompt_mm_bench.py"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2603_05353_b200 import _native as N  # noqa: E402
from paper_2603_05353_b200 import engine as E  # noqa: E402


def timed(fn, it=40):
    for i in range(4):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(it):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


def main():
    P, R = 3, 32
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for K, Nn in [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096)]:
        copies = max(2, int(600e6 // (K * Nn * 2)))
        Ws = [torch.randn(K, Nn, device="cuda", dtype=torch.bfloat16) for _ in range(copies)]
        x = torch.randn(P, R, K, device="cuda", dtype=torch.bfloat16)
        gb = K * Nn * 2 / 1e9
        t_cub = timed(lambda i: torch.mm(x.view(P * R, K), Ws[i % copies], out_dtype=torch.float32))
        line = f"K={K:5d} N={Nn:5d}: cuBLAS {t_cub:6.1f} us ({gb / t_cub * 1e6:5.0f} GB/s)"
        auto = E.prompt_mm_splits(Nn, K, R, sms)
        for s in sorted({1, 2, 4, auto, 8, 12}):
            if s > K // 64:
                continue
            out = torch.empty((s, R, Nn), dtype=torch.float32, device="cuda")

            def f(i, s=s, out=out):
                N.call("ifkv_prompt_mm", N.ptr(x), P, R, K, N.ptr(Ws[i % copies]), Nn, s, N.ptr(out), N.stream_handle())

            t = timed(f)
            line += f" | s={s}{'*' if s == auto else ''} {t:6.1f} us ({gb / t * 1e6:5.0f})"
        print(line, flush=True)


if __name__ == "__main__":
    main()
