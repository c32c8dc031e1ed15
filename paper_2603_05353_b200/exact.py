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
torch (cuBLAS DGEMM) and the float64 attention through torch matmuls, ~2 ms
per layer at Llama-3-8B width over 32K keys (scripts: tests/test_gpu_headline.py).
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


def prompt_scores_f64(weights, slab_k, slab_v, token_ids, positions, segments, capture_layer: int,
                      n_rows: Optional[int] = None):
    """Column scores of one prompt run at ``capture_layer`` in float64.

    slab_k / slab_v: [L][rows][Hkv][Dh] (bf16 or fp32, read exactly); the
    context is the slab rows of ``segments`` (row0, n, delta) in order, each
    key read as R(delta) k_stored (its assigned position).  Returns float64
    [n_rows] indexed by slab row (rows outside the segments stay 0), like
    ``prompt_forward(...).scores``."""
    torch = _torch()
    cfg = weights.config
    if not 0 <= capture_layer < cfg.n_layers:
        raise ConfigurationError(f"capture layer {capture_layer} outside [0, {cfg.n_layers})")
    dev = weights.device
    H, Hkv, Dh, d = cfg.n_heads, cfg.kv_heads, cfg.d_head, cfg.d_model
    G = H // Hkv
    f64 = torch.float64
    tok = token_ids if isinstance(token_ids, torch.Tensor) else torch.as_tensor(np.asarray(token_ids, np.int64))
    tok = tok.to(device=dev, dtype=torch.int64).reshape(-1)
    M = int(tok.numel())
    pos = torch.as_tensor(np.asarray(positions, np.int64), device=dev)
    if pos.numel() != M:
        raise ConfigurationError("prompt positions must match the prompt length")
    theta = torch.as_tensor(float(cfg.rope_base) ** (-2.0 * np.arange(Dh // 2, dtype=np.float64) / Dh), device=dev)
    rows = np.concatenate([r0 + np.arange(n, dtype=np.int64) for r0, n, _ in segments]) if segments else \
        np.zeros(0, np.int64)
    deltas = np.concatenate([np.full(n, dl, np.int64) for _, n, dl in segments]) if segments else np.zeros(0, np.int64)
    rows_t = torch.as_tensor(rows, device=dev)
    deltas_t = torch.as_tensor(deltas, device=dev)
    N = int(rows.size)
    n_rows = int(slab_k.shape[1]) if n_rows is None else int(n_rows)
    # prompt row t sees the whole context plus prompt rows 0..t (model.py:352-360)
    allowed = torch.ones((M, N + M), dtype=torch.bool, device=dev)
    allowed[:, N:] = torch.tril(torch.ones((M, M), dtype=torch.bool, device=dev))
    scale = math.sqrt(Dh)
    h = weights.embedding[tok].to(f64)
    for li in range(capture_layer + 1):
        lw = weights.layers[li]
        x = _rms(h, lw.attn_norm.to(f64))
        qkv = x @ lw.wqkv.to(f64).t()
        q = _rope(qkv[:, :H * Dh].reshape(M, H, Dh), pos, theta)
        k = _rope(qkv[:, H * Dh:(H + Hkv) * Dh].reshape(M, Hkv, Dh), pos, theta)
        v = qkv[:, (H + Hkv) * Dh:].reshape(M, Hkv, Dh)
        kc = slab_k[li].index_select(0, rows_t).to(f64)
        if bool((deltas_t != 0).any()):
            kc = _rope(kc, deltas_t, theta)
        all_k = torch.cat([kc, k], dim=0)
        all_v = torch.cat([slab_v[li].index_select(0, rows_t).to(f64), v], dim=0)
        capture = li == capture_layer
        ctx = torch.empty((M, H, Dh), dtype=f64, device=dev)
        col = torch.zeros(N, dtype=f64, device=dev) if capture else None
        for g in range(Hkv):
            qg = q[:, g * G:(g + 1) * G, :].permute(1, 0, 2)  # [G, M, Dh]
            logits = (qg @ all_k[:, g, :].t()) / scale  # [G, M, N + M]
            logits = torch.where(allowed[None], logits, torch.tensor(float("-inf"), dtype=f64, device=dev))
            e = torch.exp(logits - logits.amax(dim=-1, keepdim=True))
            e = torch.where(allowed[None], e, torch.zeros((), dtype=f64, device=dev))
            p = e / e.sum(dim=-1, keepdim=True)
            ctx[:, g * G:(g + 1) * G, :] = (p @ all_v[:, g, :]).permute(1, 0, 2)
            if capture:
                col += p[:, :, :N].sum(dim=(0, 1))
        if capture:
            scores = torch.zeros(n_rows, dtype=f64, device=dev)
            scores[rows_t] = col / H  # head mean, prompt-row sum (selection.py:108-124)
            return scores
        h = h + ctx.reshape(M, d) @ lw.wo.to(f64).t()
        x2 = _rms(h, lw.mlp_norm.to(f64))
        gu = x2 @ lw.wgu.to(f64).t()  # [M, 2 d_ff], gate / up interleaved in gu_block columns
        blk = weights.gu_block
        gu = gu.reshape(M, cfg.d_ff // blk, 2, blk)
        a = _silu(gu[:, :, 0, :].reshape(M, cfg.d_ff)) * gu[:, :, 1, :].reshape(M, cfg.d_ff)
        h = h + a @ lw.wdown.to(f64).t()
    raise AssertionError("unreachable")
