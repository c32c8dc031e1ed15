"""One recompute-attention launch at the C2 shape inside cudaProfilerStart/Stop
(for ncu --profile-from-start off).  Usage: python tools/attn_prof.py [lib] [gen]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200 import _native as N  # noqa: E402

lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_2603_05353_b200/_build/libifkv.so")
os.environ["IFKV_ATTN_GEN"] = sys.argv[2] if len(sys.argv) > 2 else "5"
N.load(Path(lib))
from paper_2603_05353_b200 import engine as E  # noqa: E402

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
torch.cuda.cudart().cudaProfilerStart()
E.recompute_attn(q, kk, vv, hz, H, Hkv, 128, out=out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
