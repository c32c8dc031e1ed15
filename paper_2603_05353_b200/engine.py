"""Device engine: typed wrappers over the C ABI plus the two layer loops the
path is built from.

* ``prompt_forward`` -- M prompt rows (one or many query groups) run forward
  on top of an injected, per-row-rotated KV prefix, fp32-accurate end to end
  (selection.py:127-169 via model.py:379-462).  bf16 weights are exact
  tensor-core operands; fp32 activations enter GEMMs as three bf16 terms
  (hi + mid + lo) whose fp32 products are summed, so the prompt forward is
  fp32-accurate and the selected set matches the float64 reference.
* ``layer_stack`` -- S tokens advance through every layer, their fresh K/V
  scattered into a slab in place before the layer's attention reads it
  (recompute.py:67-122; the same loop prefills chunks, cache.py:74-99).

PyTorch is plumbing here: tensors own HBM and the current stream orders
work.  Every bf16 step is an sm_100a kernel behind include/ifkv.h (the
projection GEMMs included: csrc/tc_gemm.cu); only the fp32 parity mode's
GEMMs use torch.mm.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .errors import ConfigurationError

ITEM_KEYS = 128  # keys per prompt-attention work item (<= kItemKeysMax)
PROMPT_ITEM_KEYS = 128  # prompt keys per causal prompt item
MERGE_ROWS_MAX_ITEMS = int(os.environ.get("IFKV_MERGE_ROWS_MAX_ITEMS", "8"))  # warp-per-row merge up to this many

# Optional CUDA-event brackets around named kernels: {name: [(start, end, work)]}
# (the benchmark sets this to measure per-launch durations for the roofline).
PROFILE = None


class _Bracket:
    def __init__(self, name, work=None):
        self.name, self.work = name, work

    def __enter__(self):
        if PROFILE is not None:
            torch = _torch()
            self.ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            self.ev[0].record()
        return self

    def __exit__(self, *exc):
        if PROFILE is not None:
            self.ev[1].record()
            PROFILE.setdefault(self.name, []).append((self.ev[0], self.ev[1], self.work))
        return False


def _torch():
    import torch

    return torch


def dt_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.bfloat16:
        return N.IFKV_BF16
    if t.dtype == torch.float32:
        return N.IFKV_F32
    raise ConfigurationError(f"unsupported tensor dtype {t.dtype}")


def _s():
    return N.stream_handle()



# ---------------------------------------------------------------------------
# thin wrappers
# ---------------------------------------------------------------------------


# CUDA-graph support (pipeline.QueryGraph): while H2D_CACHE is a dict, h2d
# returns one device copy per distinct host content (the query's static
# metadata: rows, work items, positions are uploaded once and the captured
# graph reads them in place, with no host copy inside it); while CAPTURING, a
# content that was not seen in the warm-up run is an error (a per-query host
# input must reach a captured graph through a static device buffer).
H2D_CACHE = None
CAPTURING = False


def h2d(a, device, dtype=None):
    """Host array -> device tensor through a pinned staging buffer with a
    non-blocking copy: the host never waits on the stream (pageable copies
    can), so it keeps running ahead of the GPU.  The caching host allocator
    does not reuse the staging buffer before the copy has completed."""
    torch = _torch()
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    if H2D_CACHE is not None:
        key = (arr.dtype.str, arr.shape, arr.tobytes(), str(device))
        hit = H2D_CACHE.get(key)
        if hit is not None:
            return hit
        if CAPTURING:
            raise RuntimeError("host data that differs from the warm-up run reached a CUDA-graph capture")
    if arr.size == 0:
        out = torch.from_numpy(arr).to(device)
    else:
        out = torch.from_numpy(arr).pin_memory().to(device, non_blocking=True)
    if H2D_CACHE is not None:
        H2D_CACHE[key] = out
    return out


def to_device_i64(a, device):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int64)
    return h2d(a, device, np.int64)


def rope_table(positions, d_head: int, base: float, device) -> "object":
    """fp32 (cos, sin) table [n, d_head/2, 2], angles in fp64 on device."""
    torch = _torch()
    pos = to_device_i64(positions, device).contiguous()
    cs = torch.empty((pos.numel(), d_head // 2, 2), dtype=torch.float32, device=device)
    N.call("ifkv_rope_table", N.ptr(pos), pos.numel(), d_head, float(base), N.ptr(cs), _s())
    return cs


def rotate_rows(src, dst, row_table, cs):
    """Kernel 1 over [L, T, Hkv, Dh] slabs (dst may be src: in place)."""
    L, T, Hkv, Dh = src.shape
    if T == 0:
        return dst
    N.call("ifkv_rotate_rows", dt_code(src), N.ptr(src), N.ptr(dst), src.stride(0), L, T, Hkv, Dh,
           N.ptr(row_table), N.ptr(cs), _s())
    return dst


def assemble_gather(src_keys: Sequence, src_values: Sequence, dst_k, dst_v, row0: Sequence[int], cs_row=None,
                    cs=None):
    """Gather chunk K/V into slab rows row0[c] ..; with ``cs_row``/``cs``
    (per-chunk row of a (cos, sin) table, -1 = none) the keys are rotated
    while copied (ifkv_assemble_gather_rotate)."""
    import ctypes as C

    n = len(src_keys)
    if n == 0:
        return
    L, _, Hkv, Dh = dst_k.shape
    pk = (C.c_void_p * n)(*[t.data_ptr() for t in src_keys])
    pv = (C.c_void_p * n)(*[t.data_ptr() for t in src_values])
    strides = (C.c_int64 * n)(*[t.stride(0) for t in src_keys])
    lens = (C.c_int32 * n)(*[t.shape[1] for t in src_keys])
    r0 = (C.c_int32 * n)(*[int(r) for r in row0])
    for tk, tv in zip(src_keys, src_values):
        for t in (tk, tv):
            if (t.stride(3), t.stride(2), t.stride(1)) != (1, Dh, Hkv * Dh) or t.dtype != dst_k.dtype:
                raise ConfigurationError("chunk KV rows must be contiguous [L, len, Hkv, Dh] of the slab dtype")
        if tk.stride(0) != tv.stride(0):
            raise ConfigurationError("chunk keys and values must share a layer stride")
    if cs_row is None:
        N.call("ifkv_assemble_gather", dt_code(dst_k), n, C.cast(pk, C.c_void_p), C.cast(pv, C.c_void_p),
               C.cast(strides, C.c_void_p), C.cast(lens, C.c_void_p), C.cast(r0, C.c_void_p), N.ptr(dst_k),
               N.ptr(dst_v), dst_k.stride(0), L, Hkv * Dh, _s())
        return
    crow = (C.c_int32 * n)(*[int(x) for x in cs_row])
    with _Bracket("assemble_rotate", 4 * sum(t.shape[1] for t in src_keys) * L * Hkv * Dh * dst_k.element_size()):
        N.call("ifkv_assemble_gather_rotate", dt_code(dst_k), n, C.cast(pk, C.c_void_p), C.cast(pv, C.c_void_p),
               C.cast(strides, C.c_void_p), C.cast(lens, C.c_void_p), C.cast(r0, C.c_void_p),
               C.cast(crow, C.c_void_p), N.ptr(cs), Dh, N.ptr(dst_k), N.ptr(dst_v), dst_k.stride(0), L, Hkv * Dh,
               _s())


def add_rmsnorm(h, delta, n_parts: int, gain, out_mode: int):
    torch = _torch()
    rows, d = h.shape
    out = None
    if out_mode == N.OUT_F32:
        out = torch.empty((rows, d), dtype=torch.float32, device=h.device)
    elif out_mode == N.OUT_BF16:
        out = torch.empty((rows, d), dtype=torch.bfloat16, device=h.device)
    elif out_mode == N.OUT_SPLIT3:
        out = torch.empty((3, rows, d), dtype=torch.bfloat16, device=h.device)
    ddt = dt_code(delta) if delta is not None else N.IFKV_F32
    N.call("ifkv_add_rmsnorm", N.ptr(h), N.ptr(delta), ddt, n_parts if delta is not None else 0, N.ptr(gain),
           rows, d, out_mode, N.ptr(out), _s())
    return out


def residual_add(h, delta, n_parts: int):
    N.call("ifkv_add_rmsnorm", N.ptr(h), N.ptr(delta), dt_code(delta), n_parts, None, h.shape[0], h.shape[1],
           N.OUT_F32, None, _s())


def silu_mul(gu, n_parts: int, d_ff: int, out_mode: int, gu_block: int):
    """gu [n_parts, rows, 2 d_ff] (gate/up interleaved in gu_block blocks)."""
    torch = _torch()
    rows = gu.shape[-2]
    shape = (3, rows, d_ff) if out_mode == N.OUT_SPLIT3 else (rows, d_ff)
    dt = torch.float32 if out_mode == N.OUT_F32 else torch.bfloat16
    out = torch.empty(shape, dtype=dt, device=gu.device)
    N.call("ifkv_silu_mul", N.ptr(gu), dt_code(gu), n_parts, rows, d_ff, gu_block, out_mode, N.ptr(out), _s())
    return out


def embed_rows(table, ids):
    torch = _torch()
    ids = ids.contiguous()
    h = torch.empty((ids.numel(), table.shape[1]), dtype=torch.float32, device=table.device)
    N.call("ifkv_embed_rows", N.ptr(table), dt_code(table), N.ptr(ids), ids.numel(), table.shape[1], N.ptr(h), _s())
    return h


def row_dist_accum(a, b, acc):
    """acc[r] += || a[r] - b[r] ||_2 over fp32 [rows, d] (fp64 accumulator)."""
    rows, d = a.shape
    N.call("ifkv_row_dist_accum", N.ptr(a), N.ptr(b), rows, d, N.ptr(acc), _s())


def split3(x):
    torch = _torch()
    out = torch.empty((3,) + tuple(x.shape), dtype=torch.bfloat16, device=x.device)
    N.call("ifkv_split3", N.ptr(x), x.numel(), N.ptr(out), _s())
    return out


def qkv_rope_scatter(qkv, n_parts, H, Hkv, Dh, cs, q_out, k_dst, v_dst, dst_rows):
    rows = qkv.shape[-2]
    out_dt = dt_code(k_dst)
    N.call("ifkv_qkv_rope_scatter", N.ptr(qkv), dt_code(qkv), n_parts, rows, H, Hkv, Dh, N.ptr(cs), out_dt,
           N.ptr(q_out), N.ptr(k_dst), N.ptr(v_dst), N.ptr(dst_rows), _s())


def topk_segments(scores, seg_begin, seg_k, agg_mode: int = N.AGG_NONE):
    """Segmented exact top-k; seg_begin/seg_k are host int sequences."""
    torch = _torch()
    dev = scores.device
    seg_begin = np.asarray(seg_begin, dtype=np.int32)
    seg_k = np.asarray(seg_k, dtype=np.int32)
    out_begin = np.concatenate([[0], np.cumsum(seg_k)]).astype(np.int32)
    meta = h2d(np.concatenate([seg_begin, seg_k, out_begin]), dev)
    nseg = seg_k.size
    out = torch.empty(int(out_begin[-1]), dtype=torch.int64, device=dev)
    agg = torch.empty(nseg, dtype=torch.float64, device=dev) if agg_mode != N.AGG_NONE else None
    base = meta.data_ptr()
    N.call("ifkv_topk_segments", N.ptr(scores), base, base + 4 * (nseg + 1), base + 4 * (2 * nseg + 1), nseg,
           N.ptr(out), agg_mode, N.ptr(agg), _s())
    return out, agg, out_begin


def recompute_attn_partial(q, k_layer, v_layer, horizon, H, Hkv, Dh):
    """Attention of q over this shard's keys only: (normalised ctx, ml [S,H,2])."""
    torch = _torch()
    S = q.shape[0]
    out = torch.empty_like(q)
    ml = torch.empty((S, H, 2), dtype=torch.float32, device=q.device)
    if S:
        N.call("ifkv_recompute_attn_partial", dt_code(q), N.ptr(q), N.ptr(k_layer), N.ptr(v_layer), N.ptr(horizon),
               S, H, Hkv, Dh, k_layer.shape[0], 1.0 / math.sqrt(Dh), N.ptr(out), N.ptr(ml), _s())
    return out, ml


def merge_partials(parts_o, parts_ml):
    """parts_o bf16 [P, S, H, Dh] (each normalised), parts_ml fp32 [P, S, H, 2]
    -> merged bf16 [S, H, Dh] (ifkv_merge_partials, fixed part order)."""
    torch = _torch()
    P, S, H, Dh = parts_o.shape
    out = torch.empty((S, H, Dh), dtype=parts_o.dtype, device=parts_o.device)
    N.call("ifkv_merge_partials", N.ptr(parts_o.contiguous()), N.ptr(parts_ml.contiguous()), P, S * H, Dh, N.ptr(out),
           None, _s())
    return out


def merge_prompt_states(parts_ctx, parts_ml):
    """parts_ctx fp32 [P, G, M, H, Dh], parts_ml fp32 [P, G, H, M, 2] -> merged
    (ctx [G, M, H, Dh], ml [G, H, M, 2]) (ifkv_merge_prompt_states)."""
    torch = _torch()
    P, G, M, H, Dh = parts_ctx.shape
    ctx = torch.empty(parts_ctx.shape[1:], dtype=torch.float32, device=parts_ctx.device)
    ml = torch.empty(parts_ml.shape[1:], dtype=torch.float32, device=parts_ctx.device)
    N.call("ifkv_merge_prompt_states", N.ptr(parts_ctx.contiguous()), N.ptr(parts_ml.contiguous()), P, G, M, H, Dh,
           N.ptr(ctx), N.ptr(ml), _s())
    return ctx, ml


def recompute_attn(q, k_layer, v_layer, horizon, H, Hkv, Dh, out=None, impl: str = "auto", key_start=None):
    """impl: "auto" (tcgen05 when supported, else SIMT) or "simt".
    ``key_start`` (device int64, optional): rows attend keys key_start..horizon."""
    torch = _torch()
    S = q.shape[0]
    if out is None:
        out = torch.empty_like(q)
    if key_start is not None:
        N.call("ifkv_recompute_attn_range", dt_code(q), N.ptr(q), N.ptr(k_layer), N.ptr(v_layer), N.ptr(key_start),
               N.ptr(horizon), S, H, Hkv, Dh, k_layer.shape[0], 1.0 / math.sqrt(Dh), N.ptr(out), _s())
        return out
    name = "ifkv_recompute_attn" if impl == "auto" else "ifkv_recompute_attn_simt"
    N.call(name, dt_code(q), N.ptr(q), N.ptr(k_layer), N.ptr(v_layer), N.ptr(horizon), S, H, Hkv, Dh,
           k_layer.shape[0], 1.0 / math.sqrt(Dh), N.ptr(out), _s())
    return out


# ---------------------------------------------------------------------------
# GEMMs (cuBLAS via torch.mm): fp32-accurate variant for the scoring path
# ---------------------------------------------------------------------------


# Scoring-pass GEMMs of the prompt rows on our tcgen05 weight-stream kernel
# (ifkv_prompt_mm) instead of cuBLAS; IFKV_PROMPT_MM=0 restores cuBLAS (A/B).
PROMPT_MM = os.environ.get("IFKV_PROMPT_MM", "1") != "0"
_SMS: List[int] = []


_SIDE: dict = {}


def _side_stream(idx: int = 0):
    """Side streams per device for work that can overlap the current
    stream's kernels (fork/join through events): 0 = the scoring pass's
    prompt items (high priority), 1 = unused, 2 = the scoring pass itself
    (high priority, so its CTAs are scheduled ahead of the rotating gather
    it overlaps)."""
    torch = _torch()
    key = (torch.cuda.current_device(), idx)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=key[0], priority=-1 if idx != 1 else 0)
    return _SIDE[key]


def _sm_count() -> int:
    if not _SMS:
        torch = _torch()
        _SMS.append(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count)
    return _SMS[0]


def prompt_mm_splits(N: int, K: int, R: int, sms: int, P: int = 3) -> int:
    """K splits of ifkv_prompt_mm: as many (n-tile, split) CTAs as fit in ONE
    wave (a second, partial wave of a weight stream costs more than the
    split partials; measured in tools/prompt_mm_bench.py), >= 2 k-steps each."""
    n_tiles, k_steps = N // 128, K // 64
    per_sm = 2 if 3 * (16384 + P * R * 128) + 2048 <= 113 * 1024 else 1  # 3-stage ring per CTA
    if os.environ.get("IFKV_PMM_PER_SM"):  # A/B override (with a library built for another ring depth)
        per_sm = int(os.environ["IFKV_PMM_PER_SM"])
    return max(1, min((per_sm * sms) // n_tiles, k_steps // 2))


def prompt_mm_ok(x, w) -> bool:
    torch = _torch()
    if not (PROMPT_MM and x.dim() == 3 and x.dtype == torch.bfloat16 and w.dtype == torch.bfloat16):
        return False
    p, rows, k = x.shape
    return (rows % 32 == 0 and p * rows <= 256 and k % 64 == 0 and w.shape[1] == k and w.shape[0] % 128 == 0
            and x.is_contiguous() and w.is_contiguous())


# Projection GEMMs (C = A W^T, weights stored "out x in"): bf16 operands run
# on the tcgen05 CTA-pair GEMM (ifkv_gemm*, csrc/tc_gemm.cu) with the
# consumer fused into its epilogue; fp32 operands (the fp32 parity mode) use
# torch.mm.  IFKV_GEMM_TILE overrides the tile choice (A/B: 1000 + BN).
GEMM_TILE = int(os.environ.get("IFKV_GEMM_TILE", "0"))


def _gemm_flops(m, k, n):
    return 2 * m * k * n


def gemm(a, w, out_dtype=None, out=None, accumulate: bool = False):
    """a [M, K] @ w[N, K]^T -> [M, N] (bf16 or fp32); accumulate adds into
    ``out`` (fp32).  fp32 operands go through torch.mm."""
    torch = _torch()
    M, K = a.shape
    n = w.shape[0]
    if a.dtype == torch.float32:
        if accumulate:
            out.addmm_(a, w.t())
            return out
        return torch.mm(a, w.t(), out=out) if out is not None else torch.mm(a, w.t())
    if out is None:
        out = torch.empty((M, n), dtype=out_dtype or torch.bfloat16, device=a.device)
    with _Bracket("gemm", _gemm_flops(M, K, n)):
        N.call("ifkv_gemm", N.ptr(a), a.stride(0), M, K, N.ptr(w), n, dt_code(out), N.ptr(out), out.stride(0),
               1 if accumulate else 0, GEMM_TILE, _s())
    return out


def gemm_qkv_rope_scatter(x, w, H, Hkv, cs, q_out, k_dst, v_dst, dst_rows, kv_only: bool = False):
    M, K = x.shape
    with _Bracket("gemm", _gemm_flops(M, K, w.shape[0])):
        N.call("ifkv_gemm_qkv_rope_scatter", N.ptr(x), x.stride(0), M, K, N.ptr(w), H, Hkv, 1 if kv_only else 0,
               N.ptr(cs), N.ptr(q_out), N.ptr(k_dst), N.ptr(v_dst), N.ptr(dst_rows), GEMM_TILE, _s())


def gemm_swiglu(x, w, d_ff):
    torch = _torch()
    M, K = x.shape
    out = torch.empty((M, d_ff), dtype=torch.bfloat16, device=x.device)
    with _Bracket("gemm", _gemm_flops(M, K, 2 * d_ff)):
        N.call("ifkv_gemm_swiglu", N.ptr(x), x.stride(0), M, K, N.ptr(w), d_ff, N.ptr(out), GEMM_TILE, _s())
    return out


def mm_parts(x, w):
    """x: [P, rows, K] (bf16 split terms) or [rows, K] fp32; w [N, K];
    returns fp32 [n, rows, N] part blocks whose sum is x @ w^T (consumers sum
    the n blocks): exact products, fp32 sums.  Prompt-row shapes run on
    ifkv_prompt_mm (n = its K splits, the P terms summed in its epilogue),
    larger bf16 ones (the reorder first pass: K groups x 32 rows) on the
    tcgen05 GEMM with an fp32 output (n = P), fp32 ones on torch."""
    torch = _torch()
    if prompt_mm_ok(x, w):
        p, rows, k = x.shape
        n = w.shape[0]
        s = prompt_mm_splits(n, k, rows, _sm_count(), p)
        out = torch.empty((s, rows, n), dtype=torch.float32, device=x.device)
        with _Bracket("prompt_mm", k * n * 2 + p * rows * k * 2 + s * rows * n * 4):  # W + X read, partials written
            N.call("ifkv_prompt_mm", N.ptr(x), p, rows, k, N.ptr(w), n, s, N.ptr(out), _s())
        return out
    if x.dim() == 3:
        p, rows, k = x.shape
        y = gemm(x.reshape(p * rows, k), w, out_dtype=torch.float32)
        return y.view(p, rows, w.shape[0])
    return torch.mm(x, w.t()).unsqueeze(0)


# ---------------------------------------------------------------------------
# Prompt forward over an injected prefix
# ---------------------------------------------------------------------------


@dataclass
class PromptGroup:
    """One independent prompt run: its tokens/positions and the slab rows it
    attends, as runs (row0, n_rows, delta) where keys are read as
    R(delta) k_stored."""

    token_ids: np.ndarray
    positions: np.ndarray
    segments: List[Tuple[int, int, int]]


@dataclass
class PromptOut:
    scores: Optional["object"] = None  # fp32 [T] indexed by slab row (capture layer)
    logits: Optional["object"] = None  # fp32 [G, vocab] (last prompt row of each group)
    ml: Optional["object"] = None


def segments_from_rows(rows: np.ndarray, deltas: np.ndarray) -> List[Tuple[int, int, int]]:
    """Runs (row0, n, delta) of consecutive slab rows with one rotation delta
    (context token i lives in slab row rows[i])."""
    rows = np.asarray(rows, dtype=np.int64)
    deltas = np.asarray(deltas, dtype=np.int64)
    if rows.size == 0:
        return []
    cut = np.flatnonzero((np.diff(rows) != 1) | (np.diff(deltas) != 0)) + 1
    starts = np.concatenate([[0], cut])
    ends = np.concatenate([cut, [rows.size]])
    return [(int(rows[a]), int(b - a), int(deltas[a])) for a, b in zip(starts, ends)]


def segments_from_deltas(deltas: np.ndarray, row_offset: int = 0) -> List[Tuple[int, int, int]]:
    """Runs of constant rotation delta over rows row_offset + [0, len)."""
    deltas = np.asarray(deltas, dtype=np.int64)
    if deltas.size == 0:
        return []
    cut = np.flatnonzero(np.diff(deltas)) + 1
    starts = np.concatenate([[0], cut])
    ends = np.concatenate([cut, [deltas.size]])
    return [(row_offset + int(a), int(b - a), int(deltas[a])) for a, b in zip(starts, ends)]


def _plan_items(groups: Sequence[PromptGroup], M: int, item_keys: int = ITEM_KEYS):
    """Work items (24-byte ifkv_attn_item rows): every group's context items
    (<= ITEM_KEYS keys of one constant-delta run), groups in order, then each
    group's causal prompt items (its M prompt keys in blocks of <= 128, so
    any prompt length works).  Returns (items, ctx_begin [G+1], n_ctx,
    qset_group, qset_cs, deltas)."""
    deltas = sorted({d for g in groups for (_, _, d) in g.segments if d != 0})
    delta_id = {d: i for i, d in enumerate(deltas)}
    qset_group, qset_cs, qset_of = [], [], {}

    def qset(gi, d):
        key = (gi, d)
        if key not in qset_of:
            qset_of[key] = len(qset_group)
            qset_group.append(gi)
            qset_cs.append(delta_id[d] if d != 0 else -1)
        return qset_of[key]

    items, ctx_begin = [], [0]
    for gi, g in enumerate(groups):
        for row0, n, d in g.segments:
            qs = qset(gi, d)
            for off in range(0, n, item_keys):
                items.append((gi, qs, row0 + off, min(item_keys, n - off), 0, 1))
        ctx_begin.append(len(items))
    n_ctx = len(items)
    for gi in range(len(groups)):
        for k0 in range(0, M, PROMPT_ITEM_KEYS):
            items.append((gi, qset(gi, 0), k0, min(PROMPT_ITEM_KEYS, M - k0), 1, 0))
    return (np.asarray(items, dtype=np.int32).reshape(-1, 6), np.asarray(ctx_begin, np.int32), n_ctx,
            np.asarray(qset_group, np.int32), np.asarray(qset_cs, np.int32), deltas)


def _tc_item_keys(groups, Hkv: int, G: int, M: int, sms: int = 148) -> int:
    """Keys per tensor-core work item: the longest multiple of 128 (<= 16
    blocks) that still keeps >= 80 % of the SMs busy (one 224 KB CTA per SM).
    Long items amortise each CTA's setup (TMEM alloc, 96 KB of split queries)
    and leave fewer (m, l, O) partials to merge: at C2, 2048-key items take
    the scoring stage from 5.9 to 5.3-5.7 ms vs 512-key items (2 CTAs per SM)."""
    if os.environ.get("IFKV_PROMPT_ITEM_KEYS"):  # A/B override (multiple of 128)
        return int(os.environ["IFKV_PROMPT_ITEM_KEYS"])
    hpt = max(1, min(128 // M, G))
    chunks = Hkv * (-(-G // hpt))
    runs = [n for g in groups for (_, n, _) in g.segments]
    for ipc in (16, 8, 4, 2):
        ctas = chunks * sum(-(-n // (128 * ipc)) for n in runs)
        if ctas >= 0.8 * sms:
            return 128 * ipc
    return 128


def prompt_forward(weights, slab_k, slab_v, groups: Sequence[PromptGroup], capture_layer: Optional[int] = None,
                   want_logits: bool = False, impl: str = "auto", merge_hook=None,
                   include_prompt: bool = True) -> PromptOut:
    """Run every group's prompt forward; capture column scores at
    ``capture_layer`` (then stop) or return last-row logits.  impl "auto"
    uses the tcgen05 kernels for bf16 slabs with Dh = 128, "simt" forces the
    generic kernels.  Chunk sharding: ``merge_hook(ctx, ml) -> (ctx, ml)``
    merges this rank's attention state with the other ranks' after every
    layer, and ``include_prompt`` adds the prompt's own keys (one rank only)."""
    torch = _torch()
    cfg = weights.config
    dev = weights.device
    H, Hkv, Dh, d = cfg.n_heads, cfg.kv_heads, cfg.d_head, cfg.d_model
    G = len(groups)
    dev_ids = all(isinstance(g.token_ids, torch.Tensor) for g in groups)  # device prompt ids (graph replay)
    M = int(groups[0].token_ids.numel() if dev_ids else np.asarray(groups[0].token_ids).size)
    if any(int(g.token_ids.numel() if dev_ids else np.asarray(g.token_ids).size) != M for g in groups):
        raise ConfigurationError("all prompt groups must have the same length")
    bf16 = weights.precision == "bf16"
    mode = N.OUT_SPLIT3 if bf16 else N.OUT_F32
    kv_dt = dt_code(slab_k)
    use_tc = impl == "auto" and bool(N.call("ifkv_prompt_attn_tc_supported", kv_dt, H, Hkv, M, Dh))
    item_keys = _tc_item_keys(groups, Hkv, H // Hkv, M) if use_tc else ITEM_KEYS
    items_np, ctx_begin_np, n_ctx, qg_np, qc_np, deltas = _plan_items(groups, M, item_keys)
    n_items, n_qsets = items_np.shape[0], qg_np.size
    qs_list = np.argsort(qg_np, kind="stable").astype(np.int32)  # each group's query sets, contiguous
    qs_begin = np.searchsorted(qg_np[qs_list], np.arange(G + 1)).astype(np.int32)
    max_group_qsets = max(1, int(np.diff(qs_begin).max()))  # prompt_qkv's launch extent over query sets
    # merge: a warp per output row when every group has few items (a CTA per row is launch-bound there)
    merge_items = int(np.diff(ctx_begin_np).max()) + -(-M // PROMPT_ITEM_KEYS)
    merge_fn = "ifkv_prompt_attn_merge_rows" if merge_items <= MERGE_ROWS_MAX_ITEMS else "ifkv_prompt_attn_merge"
    meta = h2d(np.concatenate([items_np.ravel(), ctx_begin_np, qg_np, qc_np, qs_begin, qs_list]), dev)
    items_p = meta.data_ptr()
    prompt_items_p = items_p + 24 * n_ctx
    ib_p = items_p + 4 * items_np.size
    qg_p = ib_p + 4 * ctx_begin_np.size
    qc_p = qg_p + 4 * qg_np.size
    qsb_p = qc_p + 4 * qc_np.size
    qsl_p = qsb_p + 4 * qs_begin.size
    cs_delta = rope_table(np.asarray(deltas, np.int64) if deltas else np.zeros(1, np.int64), Dh, cfg.rope_base, dev)
    if dev_ids:
        ids = torch.cat([g.token_ids.to(device=dev, dtype=torch.int64).reshape(-1) for g in groups])
    else:
        ids = h2d(np.concatenate([np.asarray(g.token_ids, np.int64) for g in groups]), dev)
    pos_all = np.concatenate([np.asarray(g.positions, np.int64) for g in groups])
    if pos_all.min() < 0 or pos_all.max() >= cfg.max_position:
        raise ConfigurationError(f"position outside [0, {cfg.max_position}): {int(pos_all.max())}")
    if capture_layer is not None and not 0 <= capture_layer < cfg.n_layers:
        raise ConfigurationError(f"capture layer {capture_layer} outside [0, {cfg.n_layers})")
    cs_prompt = rope_table(pos_all, Dh, cfg.rope_base, dev)
    rows = G * M
    n_rows = slab_k.shape[1]
    h = embed_rows(weights.embedding, ids)
    kp = torch.empty((rows, Hkv, Dh), dtype=torch.float32, device=dev)
    vp = torch.empty_like(kp)
    qd = torch.empty((n_qsets, H, M, Dh), dtype=torch.float32, device=dev)
    qd3 = torch.empty((n_qsets, 3, H, M, Dh), dtype=torch.bfloat16, device=dev) if use_tc else None
    part_ml = torch.empty((n_items, H, M, 2), dtype=torch.float32, device=dev)
    part_o = torch.empty((n_items, H, M, Dh), dtype=torch.float32, device=dev)
    ctx = torch.empty((G, M, H, Dh), dtype=torch.float32, device=dev)
    ml = torch.empty((G, H, M, 2), dtype=torch.float32, device=dev)
    ctx3 = torch.empty((3, rows, d), dtype=torch.bfloat16, device=dev) if bf16 else None
    scale = 1.0 / math.sqrt(Dh)
    pending, pending_parts = None, 0
    last = cfg.n_layers - 1 if capture_layer is None else capture_layer
    out = PromptOut()
    stride_ml, stride_o = H * M * 2 * 4, H * M * Dh * 4
    for li in range(last + 1):
        lw = weights.layers[li]
        x = add_rmsnorm(h, pending, pending_parts, lw.attn_norm, mode)
        qkv = mm_parts(x, lw.wqkv)
        N.call("ifkv_prompt_qkv", N.ptr(qkv), qkv.shape[0], G, M, H, Hkv, Dh, N.ptr(cs_prompt), qsb_p, qsl_p, qc_p,
               max_group_qsets, N.ptr(cs_delta), N.ptr(kp), N.ptr(vp), N.ptr(qd), N.ptr(qd3), _s())
        capture = capture_layer is not None and li == capture_layer
        with _Bracket("prompt_attn", li):
            side = include_prompt and use_tc and n_ctx and torch.cuda.is_available()
            if side:  # the prompt's own keys (SIMT) on the SMs the tensor-core grid leaves idle
                fork = torch.cuda.Event()
                fork.record()
                side_stream = _side_stream()
                side_stream.wait_event(fork)
                with torch.cuda.stream(side_stream):
                    N.call("ifkv_prompt_attn_partial", kv_dt, N.ptr(qd), N.ptr(slab_k[li]), N.ptr(slab_v[li]),
                           N.ptr(kp), N.ptr(vp), prompt_items_p, n_items - n_ctx, min(M, PROMPT_ITEM_KEYS), H, Hkv,
                           M, Dh, scale, part_ml.data_ptr() + n_ctx * stride_ml,
                           part_o.data_ptr() + n_ctx * stride_o, _s())
                    join = torch.cuda.Event()
                    join.record()
            if use_tc and n_ctx:
                N.call("ifkv_prompt_attn_partial_tc", N.ptr(qd3), n_qsets, N.ptr(slab_k[li]), N.ptr(slab_v[li]),
                       n_rows, items_p, n_ctx, item_keys, H, Hkv, M, scale, N.ptr(part_ml), N.ptr(part_o), _s())
            elif n_ctx:
                N.call("ifkv_prompt_attn_partial", kv_dt, N.ptr(qd), N.ptr(slab_k[li]), N.ptr(slab_v[li]), N.ptr(kp),
                       N.ptr(vp), items_p, n_ctx, item_keys, H, Hkv, M, Dh, scale, N.ptr(part_ml), N.ptr(part_o),
                       _s())
            if side:
                torch.cuda.current_stream().wait_event(join)
            elif include_prompt:
                N.call("ifkv_prompt_attn_partial", kv_dt, N.ptr(qd), N.ptr(slab_k[li]), N.ptr(slab_v[li]), N.ptr(kp),
                       N.ptr(vp), prompt_items_p, n_items - n_ctx, min(M, PROMPT_ITEM_KEYS), H, Hkv, M, Dh, scale,
                       part_ml.data_ptr() + n_ctx * stride_ml, part_o.data_ptr() + n_ctx * stride_o, _s())
            fuse_split = bf16 and merge_hook is None and not capture
            N.call(merge_fn, N.ptr(part_ml), N.ptr(part_o), ib_p, n_ctx if include_prompt else -1,
                   -(-M // PROMPT_ITEM_KEYS), G,
                   H, M, Dh, N.ptr(ctx), N.ptr(ml), N.ptr(ctx3) if fuse_split else None, _s())
            if merge_hook is not None:
                ctx_m, ml_m = merge_hook(ctx, ml)
                ctx.copy_(ctx_m)
                ml.copy_(ml_m)
        if capture:
            scores = torch.zeros(n_rows, dtype=torch.float32, device=dev)
            with _Bracket("score_columns", li):
                if not n_ctx:
                    pass
                elif use_tc:
                    hpt = min(128 // M, H // Hkv)
                    n_chunks = Hkv * (-(-(H // Hkv) // hpt))
                    ws = torch.empty((n_ctx, n_chunks, item_keys), dtype=torch.float32, device=dev)
                    N.call("ifkv_score_columns_tc", N.ptr(qd3), n_qsets, N.ptr(slab_k[li]), n_rows, items_p, n_ctx,
                           item_keys, N.ptr(ml), H, Hkv, M, scale, N.ptr(ws), N.ptr(scores), _s())
                else:
                    N.call("ifkv_score_columns", kv_dt, N.ptr(qd), N.ptr(slab_k[li]), items_p, n_ctx, N.ptr(ml), H,
                           Hkv, M, Dh, scale, N.ptr(scores), _s())
            out.scores, out.ml = scores, ml
            return out
        if fuse_split:
            cx = ctx3
        else:
            cx = split3(ctx.view(rows, d)) if bf16 else ctx.view(rows, d)
        o = mm_parts(cx, lw.wo)
        x2 = add_rmsnorm(h, o, o.shape[0], lw.mlp_norm, mode)
        gu = mm_parts(x2, lw.wgu)
        a = silu_mul(gu, gu.shape[0], cfg.d_ff, mode, weights.gu_block)
        pending = mm_parts(a, lw.wdown)
        pending_parts = pending.shape[0]
    if want_logits:
        fin = add_rmsnorm(h, pending, pending_parts, weights.final_norm, mode)
        last_rows = fin[..., M - 1::M, :] if bf16 else fin[M - 1::M]
        out.logits = mm_parts(last_rows.contiguous(), weights.out_head).sum(0)
    return out


# ---------------------------------------------------------------------------
# Layer stack for S tokens with in-place K/V scatter (recompute / prefill)
# ---------------------------------------------------------------------------


def layer_stack(weights, token_ids, positions, k_slab, v_slab, dst_rows, horizon, want_hidden: bool = False,
                attn_fn=None, n_layers: Optional[int] = None, on_hidden=None, key_start=None):
    """Advance S tokens (device int64 ids/positions) through every layer
    (or the first ``n_layers``).

    Layer l: x = rms_norm(h); q,k,v = x W; rope at ``positions``; k,v written
    to slab rows ``dst_rows`` (so later tokens see them); attention of q over
    slab keys 0..horizon[i] (key_start[i]..horizon[i] when given: the
    block-diagonal mask of the batched chunk prefill); residual O-proj and
    MLP.  The last layer stops
    after its K/V (nothing else can change a K/V row) unless the hidden state
    is wanted; ``on_hidden(l, h)`` sees each layer's block output (fp32 [S, d],
    model.py:450-452).

    bf16 weights: four tcgen05 GEMM launches per layer with fused epilogues
    (QKV -> RoPE + in-place K/V scatter; h += ctx Wo; gate|up -> SwiGLU;
    h += a Wdown), plus RMSNorm and the attention.  fp32 weights (parity
    mode): torch.mm GEMMs with the same elementwise kernels.
    """
    torch = _torch()
    cfg = weights.config
    dev = weights.device
    H, Hkv, Dh, d = cfg.n_heads, cfg.kv_heads, cfg.d_head, cfg.d_model
    S = int(token_ids.numel())
    if S == 0 and attn_fn is None:
        return None  # (sharded ranks keep looping: every layer has collectives)
    bf16 = weights.precision == "bf16"
    act_mode = N.OUT_BF16 if bf16 else N.OUT_F32
    run = cfg.n_layers if n_layers is None else int(n_layers)
    if not 1 <= run <= cfg.n_layers:
        raise ConfigurationError(f"n_layers {run} outside [1, {cfg.n_layers}]")
    fused_qkv = bf16 and Dh == 128
    fused_mlp = bf16 and weights.gu_block == 64
    cs = rope_table(positions, Dh, cfg.rope_base, dev)
    h = embed_rows(weights.embedding, token_ids)
    qbuf = torch.empty((S, H, Dh), dtype=weights.torch_dtype, device=dev)
    attn_out = torch.empty_like(qbuf)
    for li in range(run):
        lw = weights.layers[li]
        final = li == cfg.n_layers - 1 and not want_hidden and on_hidden is None
        x = add_rmsnorm(h, None, 0, lw.attn_norm, act_mode)
        wkv = lw.wqkv[H * Dh:] if final else lw.wqkv  # the last layer only contributes K/V
        if fused_qkv:
            gemm_qkv_rope_scatter(x, wkv, H, Hkv, cs, None if final else qbuf, k_slab[li], v_slab[li], dst_rows,
                                  kv_only=final)
        else:
            qkv = gemm(x, wkv)
            with _Bracket("qkv_rope_scatter", S * wkv.shape[0] * 2 * qkv.element_size()):
                qkv_rope_scatter(qkv, 1, 0 if final else H, Hkv, Dh, cs, None if final else qbuf, k_slab[li],
                                 v_slab[li], dst_rows)
        if final:
            return None
        if attn_fn is not None:  # chunk-sharded: attention over every rank's keys
            attn_out = attn_fn(li, qbuf, k_slab[li], v_slab[li])
        else:
            with _Bracket("recompute_attn", li):
                recompute_attn(qbuf, k_slab[li], v_slab[li], horizon, H, Hkv, Dh, out=attn_out, key_start=key_start)
        gemm(attn_out.view(S, d), lw.wo, out=h, accumulate=True)  # h += ctx Wo
        x2 = add_rmsnorm(h, None, 0, lw.mlp_norm, act_mode)
        if fused_mlp:
            a = gemm_swiglu(x2, lw.wgu, cfg.d_ff)
        else:
            a = silu_mul(gemm(x2, lw.wgu).unsqueeze(0), 1, cfg.d_ff, act_mode, weights.gu_block)
        gemm(a, lw.wdown, out=h, accumulate=True)  # h += a Wdown
        if on_hidden is not None:
            on_hidden(li, h)
    return h
