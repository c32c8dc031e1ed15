"""Float64 attention-norm scoring on the GPU (``SelectionConfig(
score_precision="fp64")``).

The default scorer is fp32-accurate (every tensor-core product exact, every
sum fp32): 2-5e-6 relative score error against the float64 reference, enough
to reproduce the reference's selected set wherever the score gap at the k-th
boundary exceeds that error.  Random-init scores at 32K context put some
boundary pairs closer than fp32 resolves; the reference
orders those by float64 digits.  This module recomputes the scoring pass in
float64 -- the prompt forward up to the capture layer with every context key
moved to its assigned position, softmax attention over the full prefix, and
the head-mean / prompt-row-sum column scores -- the arithmetic of
selection.py:127-169 / model.py:278-315,379-462 at the reference's precision,
so the selected set matches the reference's float64 argsort at any margin.

It is a precision mode, not the fast path: float64 projections go through
torch (cuBLAS DGEMM) and the float64 attention through torch matmuls -- ~95 ms
per selection at the C2 shape (20 scoring layers over 32K keys) against 4 ms
for the fp32-accurate scorer (tools/fp64_select_time.py).  The reorder first
pass (reorder.py) batches its K prompt groups' projections into one GEMM.
"""

from __future__ import annotations

import math
from typing import Optional

import numpy as np

from .errors import ConfigurationError

RMS_EPS = 1e-6  # model.py:33 (the reference's rms_norm epsilon)


def _torch():
    import torch

    return torch


def _rope(x, positions, theta):
    """Rotate interleaved pairs of x [T, heads, Dh] by positions [T] * theta
    (model.py:254-270), float64 angles and trig."""
    torch = _torch()
    ang = positions.to(torch.float64)[:, None, None] * theta[None, None, :]
    c, s = torch.cos(ang), torch.sin(ang)
    even, odd = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = even * c - odd * s
    out[..., 1::2] = even * s + odd * c
    return out


def _rms(x, gain):
    torch = _torch()
    return x / torch.sqrt((x * x).mean(dim=-1, keepdim=True) + RMS_EPS) * gain


def _silu(x):
    """Overflow-free x * sigmoid(x) (model.py:283-290)."""
    torch = _torch()
    z = torch.exp(-x.abs())
    return torch.where(x < 0, x * z / (1.0 + z), x / (1.0 + z))


def prompt_scores_f64(weights, slab_k, slab_v, groups, capture_layer: int, n_rows: Optional[int] = None):
    """Column scores at ``capture_layer`` in float64 for independent prompt
    runs (``engine.PromptGroup``: token ids, positions, context segments).

    slab_k / slab_v: [L][rows][Hkv][Dh] (bf16 or fp32, read exactly); a
    group's context is the slab rows of its segments (row0, n, delta), each
    key read as R(delta) k_stored (its assigned position); prompt row t of a
    group sees that context plus the group's prompt rows 0..t.  The groups'
    projections run as one batched float64 GEMM per weight.  Returns float64
    [n_rows] indexed by slab row (rows outside every group's segments stay 0;
    groups' segments must be disjoint), like ``prompt_forward(...).scores``."""
    torch = _torch()
    cfg = weights.config
    if not 0 <= capture_layer < cfg.n_layers:
        raise ConfigurationError(f"capture layer {capture_layer} outside [0, {cfg.n_layers})")
    if not groups:
        raise ConfigurationError("no prompt groups")
    dev = weights.device
    H, Hkv, Dh, d = cfg.n_heads, cfg.kv_heads, cfg.d_head, cfg.d_model
    G = H // Hkv
    f64 = torch.float64

    def ids_of(gr):
        t = gr.token_ids if isinstance(gr.token_ids, torch.Tensor) else torch.as_tensor(np.asarray(gr.token_ids,
                                                                                                      np.int64))
        return t.to(device=dev, dtype=torch.int64).reshape(-1)

    toks = [ids_of(gr) for gr in groups]
    M = int(toks[0].numel())
    if any(int(t.numel()) != M for t in toks):
        raise ConfigurationError("all prompt groups must have the same length")
    tok = torch.cat(toks)
    pos = torch.as_tensor(np.concatenate([np.asarray(gr.positions, np.int64) for gr in groups]), device=dev)
    if pos.numel() != tok.numel():
        raise ConfigurationError("prompt positions must match the prompt length")
    theta = torch.as_tensor(float(cfg.rope_base) ** (-2.0 * np.arange(Dh // 2, dtype=np.float64) / Dh), device=dev)
    ctx_rows, ctx_deltas = [], []
    for gr in groups:
        segs = gr.segments
        r = np.concatenate([r0 + np.arange(n, dtype=np.int64) for r0, n, _ in segs]) if segs else np.zeros(0, np.int64)
        dl = np.concatenate([np.full(n, x, np.int64) for _, n, x in segs]) if segs else np.zeros(0, np.int64)
        ctx_rows.append(torch.as_tensor(r, device=dev))
        ctx_deltas.append(torch.as_tensor(dl, device=dev))
    n_rows = int(slab_k.shape[1]) if n_rows is None else int(n_rows)
    causal = torch.tril(torch.ones((M, M), dtype=torch.bool, device=dev))
    scale = math.sqrt(Dh)
    ninf = torch.tensor(float("-inf"), dtype=f64, device=dev)
    zero = torch.zeros((), dtype=f64, device=dev)
    h = weights.embedding[tok].to(f64)
    R = h.shape[0]
    for li in range(capture_layer + 1):
        lw = weights.layers[li]
        x = _rms(h, lw.attn_norm.to(f64))
        qkv = x @ lw.wqkv.to(f64).t()
        q = _rope(qkv[:, :H * Dh].reshape(R, H, Dh), pos, theta)
        k = _rope(qkv[:, H * Dh:(H + Hkv) * Dh].reshape(R, Hkv, Dh), pos, theta)
        v = qkv[:, (H + Hkv) * Dh:].reshape(R, Hkv, Dh)
        capture = li == capture_layer
        ctx = torch.empty((R, H, Dh), dtype=f64, device=dev)
        scores = torch.zeros(n_rows, dtype=f64, device=dev) if capture else None
        for gi in range(len(groups)):
            rows_t, deltas_t = ctx_rows[gi], ctx_deltas[gi]
            N = int(rows_t.numel())
            sl = slice(gi * M, (gi + 1) * M)
            kc = slab_k[li].index_select(0, rows_t).to(f64)
            if bool((deltas_t != 0).any()):
                kc = _rope(kc, deltas_t, theta)
            all_k = torch.cat([kc, k[sl]], dim=0)
            all_v = torch.cat([slab_v[li].index_select(0, rows_t).to(f64), v[sl]], dim=0)
            allowed = torch.ones((M, N + M), dtype=torch.bool, device=dev)
            allowed[:, N:] = causal
            # all kv heads in one batched matmul: [Hkv, G*M, Dh] x [Hkv, Dh, N+M]
            qg = q[sl].reshape(M, Hkv, G, Dh).permute(1, 2, 0, 3).reshape(Hkv, G * M, Dh)
            logits = torch.bmm(qg, all_k.permute(1, 2, 0)).view(Hkv, G, M, N + M) / scale
            logits = torch.where(allowed[None, None], logits, ninf)
            e = torch.exp(logits - logits.amax(dim=-1, keepdim=True))
            e = torch.where(allowed[None, None], e, zero)
            p = e / e.sum(dim=-1, keepdim=True)
            o = torch.bmm(p.view(Hkv, G * M, N + M), all_v.permute(1, 0, 2))  # [Hkv, G*M, Dh]
            ctx[sl] = o.view(Hkv, G, M, Dh).permute(2, 0, 1, 3).reshape(M, H, Dh)
            if capture:  # head mean, prompt-row sum (selection.py:108-124)
                scores[rows_t] = p[..., :N].sum(dim=(0, 1, 2)) / H
        if capture:
            return scores
        h = h + ctx.reshape(R, d) @ lw.wo.to(f64).t()
        x2 = _rms(h, lw.mlp_norm.to(f64))
        gu = x2 @ lw.wgu.to(f64).t()  # [R, 2 d_ff], gate / up interleaved in gu_block columns
        blk = weights.gu_block
        gu = gu.reshape(R, cfg.d_ff // blk, 2, blk)
        a = _silu(gu[:, :, 0, :].reshape(R, cfg.d_ff)) * gu[:, :, 1, :].reshape(R, cfg.d_ff)
        h = h + a @ lw.wdown.to(f64).t()
    raise AssertionError("unreachable")
