"""A/B of the recompute's projection GEMMs inside the C2 step: the tcgen05
pair GEMM with fused epilogues (product) against cuBLAS (torch.mm + the
separate rope/scatter and SiLU kernels, the round-1 path), alternated step by
step in one process so both see the same clocks.  Measurement tool only: the
cuBLAS arm is monkeypatched in here and never ships in the package.

    python tools/gemm_ab.py [--steps 6] [--layers 32]
"""

import argparse
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_05353_b200 as P  # noqa: E402
from paper_2603_05353_b200 import _native as N  # noqa: E402
from paper_2603_05353_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--layers", type=int, default=32)
args = ap.parse_args()

ours = (E.gemm, E.gemm_qkv_rope_scatter, E.gemm_swiglu)


def cublas_gemm(a, w, out_dtype=None, out=None, accumulate=False):
    if accumulate:
        torch.addmm(out, a, w.t(), out_dtype=torch.float32, out=out)
        return out
    if out_dtype == torch.float32:
        return torch.mm(a, w.t(), out_dtype=torch.float32)
    return torch.mm(a, w.t())


def cublas_qkv(x, w, H, Hkv, cs, q_out, k_dst, v_dst, dst_rows, kv_only=False):
    qkv = torch.mm(x, w.t())
    E.qkv_rope_scatter(qkv, 1, 0 if kv_only else H, Hkv, 128, cs, q_out, k_dst, v_dst, dst_rows)


def cublas_swiglu(x, w, d_ff):
    return E.silu_mul(torch.mm(x, w.t()).unsqueeze(0), 1, d_ff, N.OUT_BF16, 64)


def use(kind):
    E.gemm, E.gemm_qkv_rope_scatter, E.gemm_swiglu = ours if kind == "ours" else (cublas_gemm, cublas_qkv,
                                                                                 cublas_swiglu)


cfg = P.llama3_8b_config()
if args.layers != 32:
    import dataclasses

    cfg = dataclasses.replace(cfg, n_layers=args.layers)
w = P.DeviceWeights.random(cfg, seed=7)
task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=2048, prompt_length=32,
                       vocab_size=cfg.vocab_size)
g = P.generate_task(task, 0)
kvs = [P.prefill_chunk(w, c) for c in g.chunks]
sel_cfg = P.SelectionConfig(ratio=0.15)


def step():
    return P.assemble_select_recompute(w, kvs, g.chunks, g.prompt_token_ids, sel_cfg)


res = {"ours": [], "cublas": []}
sets = {}
for kind in ("ours", "cublas"):
    use(kind)
    for _ in range(2):
        r = step()
    torch.cuda.synchronize()
    sets[kind] = (r.selection.selected_numpy(), r.cache.keys[-1].float().cpu())
for i in range(args.steps):
    for kind in ("ours", "cublas") if i % 2 == 0 else ("cublas", "ours"):
        use(kind)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = step()
        b.record()
        torch.cuda.synchronize()
        res[kind].append(a.elapsed_time(b))
        del r
use("ours")
for k, v in res.items():
    print(f"{k:7s}: median {statistics.median(v):.2f} ms  all {' '.join(f'{x:.2f}' for x in v)}")
same = (sets["ours"][0] == sets["cublas"][0]).all()
dk = (sets["ours"][1] - sets["cublas"][1]).abs().max().item() / sets["cublas"][1].abs().max().item()
print(f"selected sets equal: {same}; last-layer K rel diff ours vs cublas: {dk:.2e}")
