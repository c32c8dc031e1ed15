"""clock64 trace of one v11 attention CTA (heaviest pair, kv head 0) at the C2
shape, per 64-key sub-block.
Source: profiles/attic/tc_recompute_attn_v11.cu.txt (copy it back into csrc/, dispatch it from
recompute_attn.cu, build with -DIFKV_ATTN11_TRACE=1).
Usage: python tools/attn11_trace.py _ab/v11t/libifkv.so"""
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
raw.ifkv_attn11_trace_clear()
E.recompute_attn(q, kk, vv, hz, H, Hkv, 128, out=out)
torch.cuda.synchronize()
NS = 1024
buf = np.zeros(8 * 2 * NS, np.int64)
assert raw.ifkv_attn11_trace_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
t = buf.reshape(8, 2, NS).astype(np.float64)
nb = int(np.max(np.nonzero(t[0, 0])[0])) + 1
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
lo, hi = 8, nb - 4
print(f"sub-blocks traced: {nb}; medians over {lo}..{hi} (clk)")


def med(a):
    return float(np.nanmedian(a[lo:hi]))


for x, name in ((0, "A"), (1, "B")):
    s_obs, mx, _, pub, pv, si = (t[e, x, :nb] for e in range(6))
    print(f"tile {name}: S seen -> max {med(mx - s_obs):.0f} | max -> P published {med(pub - mx):.0f} | "
          f"P(u) published -> S(u+1) seen {med(s_obs[1:] - pub[:-1]):.0f} | period {med(np.diff(s_obs)):.0f}")
    print(f"        P published -> PV issued {med(pv - pub):.0f} | PV(u) issued -> S(u+2) issued "
          f"{med(si[2:] - pv[:-2]):.0f} | S(u) issued -> seen {med(s_obs - si):.0f}")
print("MMA warp timeline (event, clk since previous): PVwait_done(6) PV_iss(4) S_iss(5) S_done(7)")
for u in range(lo, lo + 4):
    ev = []
    for x in (0, 1):
        ev += [(f"PV{'AB'[x]}({u}) ring", t[6, x, u]), (f"PV{'AB'[x]}({u}) P", t[4, x, u]),
               (f"S{'AB'[x]}({u+2}) ring", t[5, x, u + 2]), (f"S{'AB'[x]}({u+2}) issued", t[7, x, u + 2])]
    prev = None
    for name, v in ev:
        print(f"  {name:18s} {v:9.0f} {'' if prev is None else f'+{v - prev:.0f}'}")
        prev = v
print("first sub-blocks (S_iss, S_seen, max, pub, PV_iss) A | B:")
for j in range(lo, lo + 8):
    print(f"  u={j}: A {t[5,0,j]:.0f} {t[0,0,j]:.0f} {t[1,0,j]:.0f} {t[3,0,j]:.0f} {t[4,0,j]:.0f} | "
          f"B {t[5,1,j]:.0f} {t[0,1,j]:.0f} {t[1,1,j]:.0f} {t[3,1,j]:.0f} {t[4,1,j]:.0f}")
