"""Selective KV recomputation under the global causal mask (reference
recompute.py:1-122).

B200 data flow (one call):
  1. Kernel 1 moves every context key of every layer to the global decode
     layout, in place (``to_decode_layout``; the reference re-rotates the
     non-selected rows inside each layer, recompute.py:106-109);
  2. the selected tokens restart from their embeddings and run the layer
     stack; per layer their fresh K/V are rotated and scattered into the
     slab rows in place (``ifkv_qkv_rope_scatter``) before the sparse-query
     causal attention (``ifkv_recompute_attn``) reads keys 0..own index --
     equivalent to the reference's ascending-order processing because a
     layer's fresh K/V depend only on that layer's input;
  3. row metadata marks the rows RECOMPUTED_GLOBAL at their positions.

The slab is updated in place (north star: "scatters their new K/V into the
cache in place"); the returned cache shares its tensors with the input, and
the input's metadata is updated too, so both stay self-consistent.  Untouched
rows equal the decode view of the input bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import engine as E
from .cache import AssembledCache, Provenance, to_decode_layout
from .errors import ConfigurationError


def _torch():
    import torch

    return torch


@dataclass
class RecomputePlan:
    """Rows to recompute (ascending), their RoPE positions and causal
    horizons (recompute.py:30-53).  Fields may be host arrays (validated) or
    device int64 tensors from select_topk (valid by construction)."""

    selected: "object"
    positions: "object"
    allowed_upto: "object"
    trusted: bool = False

    def __post_init__(self):
        torch = _torch()
        if self.trusted or isinstance(self.selected, torch.Tensor):
            if not (self.selected.shape == self.positions.shape == self.allowed_upto.shape):
                raise ConfigurationError("plan arrays must have equal lengths")
            return
        self.selected = np.asarray(self.selected, dtype=np.int64).ravel()
        self.positions = np.asarray(self.positions, dtype=np.int64).ravel()
        self.allowed_upto = np.asarray(self.allowed_upto, dtype=np.int64).ravel()
        if self.positions.shape != self.selected.shape or self.allowed_upto.shape != self.selected.shape:
            raise ConfigurationError("plan arrays must have equal lengths")
        if self.selected.size and np.any(np.diff(self.selected) <= 0):
            raise ConfigurationError("selected indices must be strictly ascending")
        if np.any(self.allowed_upto < self.selected):
            raise ConfigurationError("allowed-key horizon must be causal (>= own index)")
        if self.selected.size and np.any(np.diff(self.allowed_upto) < 0):
            raise ConfigurationError("allowed-key horizons must be non-decreasing")

    @property
    def size(self) -> int:
        return int(self.selected.shape[0])


def make_plan(cache: AssembledCache, selected) -> RecomputePlan:
    """Standard plan: positions = horizons = the selected indices
    (recompute.py:56-64).  A device tensor produced by select_topk (tagged:
    sorted, unique, in range by construction) is used as is with no host
    sync; any other device tensor is sorted and validated on the device with
    one deferred host check (range, duplicates), like the reference's host
    checks."""
    torch = _torch()
    if isinstance(selected, torch.Tensor) and selected.is_cuda:
        n = cache.context_length
        tag = getattr(selected, "_ifkv_valid_plan", None)
        if tag is not None and tag <= n:
            sel = selected.to(torch.int64)
            return RecomputePlan(selected=sel, positions=sel, allowed_upto=sel, trusted=True)
        sel = torch.sort(selected.reshape(-1).to(torch.int64)).values
        if sel.numel():
            bad = (sel[0] < 0) | (sel[-1] >= n)
            dup = bool((sel[1:] == sel[:-1]).any().item()) if sel.numel() > 1 else False
            if bool(bad.item()):
                raise ConfigurationError(f"selected index outside context [0, {n})")
            if dup:
                raise ConfigurationError("selected indices contain duplicates")
        return RecomputePlan(selected=sel, positions=sel, allowed_upto=sel, trusted=True)
    sel = np.sort(np.asarray(selected, dtype=np.int64).ravel())
    n = cache.context_length
    if sel.size and (sel.min() < 0 or sel.max() >= n):
        raise ConfigurationError(f"selected index outside context [0, {n})")
    if np.unique(sel).size != sel.size:
        raise ConfigurationError("selected indices contain duplicates")
    return RecomputePlan(selected=sel, positions=sel.copy(), allowed_upto=sel.copy())


def recompute_selected(weights, cache: AssembledCache, plan: RecomputePlan, readback=None) -> AssembledCache:
    """Recompute the planned rows in place and return the updated cache.

    ``readback`` (graph capture, pipeline.QueryGraph): two pinned int64 host
    tensors of the plan's size; the selected indices and positions are copied
    into them asynchronously and the host-side row metadata is left to the
    caller (no host synchronisation here)."""
    torch = _torch()
    cfg = weights.config
    n = cache.context_length
    s = plan.size
    if s == 0:
        return cache
    if cache.n_layers != cfg.n_layers:
        raise ConfigurationError("cache layer count does not match model")
    if cache.keys.dtype != weights.torch_dtype:
        raise ConfigurationError(f"cache dtype {cache.keys.dtype} does not match weights ({weights.precision})")
    dev = cache.keys.device
    if not plan.trusted:
        if plan.selected.max() >= n or plan.selected.min() < 0:
            raise ConfigurationError(f"plan index outside cache context [0, {n})")
        if np.any(plan.allowed_upto >= n):
            raise ConfigurationError("allowed-key horizon outside cache context")
    sel = E.to_device_i64(plan.selected, dev)
    pos = E.to_device_i64(plan.positions, dev)
    upto = E.to_device_i64(plan.allowed_upto, dev)
    deferred = readback is not None
    if deferred:
        for h, t in zip(readback, (sel, pos)):
            h.copy_(t, non_blocking=True)
    elif plan.trusted:  # device plan: start its copy to the host now, read it after the layer stack is queued
        readback = [torch.empty(t.shape, dtype=torch.int64, pin_memory=True) for t in (sel, pos)]
        for h, t in zip(readback, (sel, pos)):
            h.copy_(t, non_blocking=True)
        done = torch.cuda.Event()
        done.record()
    to_decode_layout(cache, cfg.rope_base)
    ids = cache.token_ids_device().index_select(0, sel)
    E.layer_stack(weights, ids, pos, cache.keys, cache.values, sel, upto)
    if deferred:
        return cache
    # row metadata (host): positions and provenance of the replaced rows
    if readback is not None:
        done.synchronize()  # waits for the selection only, not for the recompute
        sel_h, pos_h = readback[0].numpy(), readback[1].numpy()
    else:
        sel_h, pos_h = plan.selected, plan.positions
    cache.row_positions[sel_h] = pos_h
    cache.provenance[sel_h] = int(Provenance.RECOMPUTED_GLOBAL)
    return replace(cache)
