"""One small pass over every tcgen05 / TMA / mbarrier kernel (C1 path through
the store and two-pass paths, tcgen05 GEMM epilogues, recompute attention with
key ranges, prompt scorer) for compute-sanitizer:
    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_c1.py"""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_05353_b200 as P  # noqa: E402
from paper_2603_05353_b200 import _native as N  # noqa: E402
from paper_2603_05353_b200 import engine as E  # noqa: E402

cfg = P.c1_config()
dw = P.DeviceWeights.from_host(P.init_weights(cfg, 7), "bf16")
task = P.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32, vocab_size=1024)
g = P.generate_task(task, 0)
store = P.prefill_chunks(dw, g.chunks)  # batched prefill: GEMM epilogues + key-range attention
res = P.assemble_select_recompute(dw, store, g.chunks, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
plain = [P.prefill_chunk(dw, c) for c in g.chunks]
res2 = P.assemble_select_recompute(dw, plain, g.chunks, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
plan, _, _ = P.reorder_and_reselect(dw, g.chunks, g.prompt_token_ids, budget=308, prefilled=plain)
# reorder over the store slab (first pass in place: warp-per-row merge, Dh = 128 SIMT partial)
plan_s, _, _ = P.reorder_and_reselect(dw, g.chunks, g.prompt_token_ids, budget=308, prefilled=store)
assert np.array_equal(plan.permutation, plan_s.permutation)
# a larger recompute attention grid (key splits, two tiles per CTA, G = 4)
rng = np.random.default_rng(0)
q = torch.randn(600, 32, 128, device="cuda").bfloat16()
k = torch.randn(3000, 8, 128, device="cuda").bfloat16()
v = torch.randn(3000, 8, 128, device="cuda").bfloat16()
hz = torch.as_tensor(np.sort(rng.choice(3000, 600, replace=False)), device="cuda")
E.recompute_attn(q, k, v, hz, 32, 8, 128)
# GEMM tile widths and epilogues
a = torch.randn(300, 512, device="cuda").bfloat16()
w = (torch.randn(768, 512, device="cuda") / 22).bfloat16()
for tile in (1256, 1192, 1128):
    E.gemm(a, w)
    h = torch.zeros(300, 768, device="cuda")
    N.call("ifkv_gemm", a.data_ptr(), 512, 300, 512, w.data_ptr(), 768, N.IFKV_F32, h.data_ptr(), 768, 1, tile,
           N.stream_handle())
torch.cuda.synchronize()
print("sanitize pass ok:", res.selection.selected_numpy().size, res2.selection.selected_numpy().size,
      plan.permutation.tolist())
