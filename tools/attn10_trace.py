"""clock64 trace of one v10 attention CTA (the heaviest pair of kv head 0) at
the C2 shape.  Build: python tools/build_variants.py v10t=IFKV_ATTN10_TRACE=1
Usage: python tools/attn10_trace.py _ab/v10t/libifkv.so"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200 import _native as N  # noqa: E402

lib = sys.argv[1]
N.load(Path(lib))
from paper_2603_05353_b200 import engine as E  # noqa: E402

raw = ctypes.CDLL(lib)
n, k, H, Hkv = 32768, 4916, 32, 8
sel = np.sort(np.random.default_rng(0).choice(n, k, replace=False))
q = torch.randn(k, H, 128, device="cuda", dtype=torch.bfloat16)
kk = torch.randn(n, Hkv, 128, device="cuda", dtype=torch.bfloat16)
vv = torch.randn(n, Hkv, 128, device="cuda", dtype=torch.bfloat16)
hz = torch.as_tensor(sel, device="cuda")
out = torch.empty_like(q)
for _ in range(3):
    E.recompute_attn(q, kk, vv, hz, H, Hkv, 128, out=out)
torch.cuda.synchronize()
raw.ifkv_attn10_trace_clear()
E.recompute_attn(q, kk, vv, hz, H, Hkv, 128, out=out)
torch.cuda.synchronize()
buf = np.zeros(6 * 2 * 512, np.int64)
assert raw.ifkv_attn10_trace_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
t = buf.reshape(6, 2, 512).astype(np.float64)
nb = int(np.max(np.nonzero(t[0, 0])[0])) + 1
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
lo, hi = 8, nb - 4
print(f"blocks traced: {nb}; medians over blocks {lo}..{hi} (clk)")


def med(a):
    return float(np.nanmedian(a[lo:hi]))


for x, name in ((0, "A"), (1, "B")):
    s_obs, mx, ex, pub, pv, si = (t[e, x, :nb] for e in range(6))
    print(f"tile {name}: S observed -> max {med(mx - s_obs):.0f} | max -> exps done {med(ex - mx):.0f} | "
          f"exps -> P published {med(pub - ex):.0f} | softmax total {med(pub - s_obs):.0f}")
    print(f"        P published -> PV issued (MMA warp) {med(pv - pub):.0f} | PV issued -> S(j+1) issued "
          f"{med(si[1:] - pv[:-1]):.0f} | S(j+1) issued -> observed {med(s_obs[1:] - si[1:]):.0f} | "
          f"period {med(np.diff(s_obs)):.0f}")
# overlap of the two tiles' exponential phases
oa = np.array([(t[1, 0, j], t[2, 0, j]) for j in range(nb)])
ob = np.array([(t[1, 1, j], t[2, 1, j]) for j in range(nb)])
ov = []
for j in range(lo, hi):
    a0, a1 = oa[j]
    for jj in (j - 1, j, j + 1):
        b0, b1 = ob[jj]
        ov.append(max(0.0, min(a1, b1) - max(a0, b0)))
print(f"exp-phase overlap A/B per block (sum over neighbours, median): {np.median(np.array(ov).reshape(-1, 3).sum(1)):.0f} clk")
print("first blocks (A: S_obs, max, exps, pub | MMA: PV_iss, S_iss):")
for j in range(lo, lo + 6):
    print(f"  j={j}: A {t[0,0,j]:.0f} {t[1,0,j]:.0f} {t[2,0,j]:.0f} {t[3,0,j]:.0f} pv {t[4,0,j]:.0f} s {t[5,0,j]:.0f} | "
          f"B {t[0,1,j]:.0f} {t[1,1,j]:.0f} {t[2,1,j]:.0f} {t[3,1,j]:.0f} pv {t[4,1,j]:.0f} s {t[5,1,j]:.0f}")
