"""Phase timeline of one recompute-attention CTA (build with
-DIFKV_ATTN_TRACE=1).  Streams: 0/1/2 = tile A softmax (wait S, S ready, P
published), 3/4/5 = tile B, 6/7 = MMA warp (wait P, P ready)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200 import _native as N  # noqa: E402


def main(lib):
    N._lib = None
    L = N.load(Path(lib))
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(0)
    n, k, H, Hkv, Dh = 32768, 4916, 32, 8, 128
    sel = np.sort(rng.choice(n, k, replace=False))
    q = torch.randn(k, H, Dh, device="cuda", dtype=torch.bfloat16)
    kk = torch.randn(n, Hkv, Dh, device="cuda", dtype=torch.bfloat16)
    vv = torch.randn(n, Hkv, Dh, device="cuda", dtype=torch.bfloat16)
    hz = torch.as_tensor(sel, device="cuda")
    buf = (C.c_longlong * (12 * 4096))()
    cnt = (C.c_int * 12)()
    E.recompute_attn(q, kk, vv, hz, H, Hkv, Dh)
    L.ifkv_attn_trace_read(buf, cnt, 1)
    E.recompute_attn(q, kk, vv, hz, H, Hkv, Dh)
    torch.cuda.synchronize()
    L.ifkv_attn_trace_read(buf, cnt, 1)
    t = np.frombuffer(buf, dtype=np.int64).reshape(12, 4096)
    c = list(cnt)
    print("counts", c)
    t0 = min(t[i, 0] for i in range(12) if c[i])
    A = [t[i, : c[i]] - t0 for i in range(12)]
    print(f"MMA wait-for-V median {np.median(A[9] - A[8]):.0f}, wait-for-K median {np.median(A[11] - A[10]):.0f}")
    nb = min(c[0], c[3])
    wait_a = A[1][:nb] - A[0][:nb]
    work_a = A[2][:nb] - A[1][:nb]
    wait_b = A[4][:nb] - A[3][:nb]
    work_b = A[5][:nb] - A[4][:nb]
    per = np.diff(A[2][:nb])
    print(f"blocks {nb}; softmax A: wait-for-S median {np.median(wait_a):.0f} cyc, work median {np.median(work_a):.0f}")
    print(f"softmax B: wait-for-S median {np.median(wait_b):.0f}, work median {np.median(work_b):.0f}")
    print(f"block period (P_A publish to publish) median {np.median(per):.0f} cycles (ideal MMA 2048)")
    mma_wait = A[7] - A[6]
    print(f"MMA warp wait-for-P median {np.median(mma_wait):.0f} cycles (n={len(mma_wait)})")
    for j in range(5, 10):
        print(j, "A:", A[0][j], A[1][j], A[2][j], " B:", A[3][j], A[4][j], A[5][j])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "_ab/trace/libifkv.so"))
