"""One launch each of cuBLAS and ifkv_gemm (per tile code) at a recompute shape (for ncu)."""
import math, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_05353_b200 import _native as N  # noqa: E402

M, K, Nn = (int(x) for x in sys.argv[1:4])
tiles = [int(x) for x in sys.argv[4:]] or [0]
a = torch.randn(M, K, device="cuda").bfloat16()
w = (torch.randn(Nn, K, device="cuda") / math.sqrt(K)).bfloat16()
wt = w.t().contiguous()
out = torch.empty(M, Nn, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    torch.mm(a, wt)
    for tn in tiles:
        N.call("ifkv_gemm", a.data_ptr(), K, M, K, w.data_ptr(), Nn, N.IFKV_BF16, out.data_ptr(), Nn, 0, tn,
               torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
