"""Chunk KV caches, assembly and the decode layout, resident in HBM
(reference cache.py:1-450).

HBM layout: every cache is a layer-major slab ``keys[L][rows][Hkv][Dh]``
(values alike), rows contiguous (Hkv*Dh elements = 2 KB per row at
Llama-3-8B shape in bf16), so a layer view is one contiguous block the
kernels stream with 128-bit accesses.  ``keys[l]`` keeps the reference's
per-layer indexing.  Small per-row metadata (token ids, rotation positions,
provenance, chunk mapping) stays on the host as NumPy arrays, exactly as in
the reference.

Cached keys carry the rotation they were computed at (``row_positions``);
moving a row to another position is one rotation by the delta (Kernel 1,
``ifkv_rotate_rows``).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import engine as E
from .errors import ConfigurationError
from .positions import ChunkSpec


class Provenance(IntEnum):
    PREFILLED_LOCAL = 0
    RECOMPUTED_GLOBAL = 1
    FULL_PREFILL = 2


def _torch():
    import torch

    return torch


@dataclass
class ChunkKV:
    """One chunk's KV in HBM: keys/values [L, len, Hkv, Dh] (cache.py:37-71)."""

    chunk_id: str
    token_ids: np.ndarray
    keys: "object"
    values: "object"
    prefill_positions: np.ndarray
    provenance: Provenance
    model_fingerprint: int
    # set by prefill_chunks: (store_k, store_v) this chunk is a row range of,
    # and its first store row -- lets the query path score straight from the
    # store and assemble with the rotation fused (pipeline.py)
    store: Optional[tuple] = field(default=None, repr=False, compare=False)
    store_row0: int = -1

    def __post_init__(self):
        self.token_ids = np.asarray(self.token_ids, dtype=np.int64)
        self.prefill_positions = np.asarray(self.prefill_positions, dtype=np.int64)
        n = self.token_ids.size
        if self.keys.dim() != 4 or self.keys.shape != self.values.shape or self.keys.shape[0] < 1:
            raise ConfigurationError("keys and values must be matching [L, len, Hkv, Dh] tensors")
        if self.keys.shape[1] != n:
            raise ConfigurationError("KV length does not match chunk length")
        if self.prefill_positions.size != n:
            raise ConfigurationError("prefill_positions length does not match chunk length")
        if self.provenance is Provenance.PREFILLED_LOCAL and not np.array_equal(self.prefill_positions, np.arange(n)):
            raise ConfigurationError("prefilled_local caches must use positions 0..len-1")

    @property
    def length(self) -> int:
        return int(self.token_ids.size)

    @property
    def n_layers(self) -> int:
        return int(self.keys.shape[0])


@dataclass
class PromptKV:
    """Fresh prompt KV (always query-time): keys/values [L, M, Hkv, Dh]."""

    token_ids: np.ndarray
    keys: "object"
    values: "object"
    positions: np.ndarray


@dataclass
class AssembledCache:
    """Chunks concatenated in declared order, then optional prompt rows
    (cache.py:216-256).  keys/values: [L, N + M, Hkv, Dh] device slabs."""

    chunk_ids: List[str]
    chunk_lengths: List[int]
    token_ids: np.ndarray
    keys: "object"
    values: "object"
    row_positions: np.ndarray
    provenance: np.ndarray
    chunk_index: np.ndarray
    local_index: np.ndarray
    prompt_length: int
    model_fingerprint: int
    _token_ids_dev: Optional["object"] = field(default=None, repr=False, compare=False)

    @property
    def context_length(self) -> int:
        return int(self.token_ids.size - self.prompt_length)

    @property
    def total_length(self) -> int:
        return int(self.token_ids.size)

    @property
    def n_layers(self) -> int:
        return int(self.keys.shape[0])

    def mapping(self, global_index: int):
        if not 0 <= global_index < self.context_length:
            raise ConfigurationError(f"global index {global_index} outside context [0, {self.context_length})")
        return self.chunk_ids[int(self.chunk_index[global_index])], int(self.local_index[global_index])

    def token_ids_device(self):
        if self._token_ids_dev is None:
            self._token_ids_dev = E.h2d(self.token_ids, self.keys.device, np.int64)
        return self._token_ids_dev

    def in_decode_layout(self) -> bool:
        n = self.context_length
        return bool(np.array_equal(self.row_positions[:n], np.arange(n)))


def assemble(chunks: Sequence[ChunkKV], prompt_kv: Optional[PromptKV] = None) -> AssembledCache:
    """Gather chunk KVs (declared order) and an optional prompt KV into a new
    per-query slab with one ``ifkv_assemble_gather`` launch (cache.py:259-322).
    The chunk store is never modified; keys keep their stored rotation."""
    torch = _torch()
    if not chunks and prompt_kv is None:
        raise ConfigurationError("nothing to assemble: no chunks and no prompt")
    if chunks:
        fp = chunks[0].model_fingerprint
        ref = chunks[0].keys
        for c in chunks:
            if c.model_fingerprint != fp:
                raise ConfigurationError(f"chunk {c.chunk_id!r} was prefetched under a different model "
                                         f"(fingerprint {c.model_fingerprint:#x} != {fp:#x})")
            if c.n_layers != ref.shape[0] or c.keys.shape[2:] != ref.shape[2:] or c.keys.dtype != ref.dtype:
                raise ConfigurationError(f"chunk {c.chunk_id!r} KV shape mismatch")
        L, _, Hkv, Dh = ref.shape
        dtype, dev = ref.dtype, ref.device
    else:
        fp = 0
        L, _, Hkv, Dh = prompt_kv.keys.shape
        dtype, dev = prompt_kv.keys.dtype, prompt_kv.keys.device
    lens = [c.length for c in chunks]
    m = 0 if prompt_kv is None else int(np.asarray(prompt_kv.token_ids).size)
    if prompt_kv is not None and prompt_kv.keys.shape[0] != L:
        raise ConfigurationError("prompt KV layer count mismatch")
    total = sum(lens) + m
    keys = torch.empty((L, total, Hkv, Dh), dtype=dtype, device=dev)
    values = torch.empty_like(keys)
    src_k = [c.keys for c in chunks]
    src_v = [c.values for c in chunks]
    row0 = list(np.concatenate([[0], np.cumsum(lens)])[:len(lens)]) if lens else []
    if prompt_kv is not None:
        src_k.append(prompt_kv.keys.to(dtype))
        src_v.append(prompt_kv.values.to(dtype))
        row0.append(sum(lens))
    E.assemble_gather(src_k, src_v, keys, values, row0)
    parts = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    tok = [c.token_ids for c in chunks] + ([np.asarray(prompt_kv.token_ids, np.int64)] if m else [])
    pos = [c.prefill_positions for c in chunks] + ([np.asarray(prompt_kv.positions, np.int64)] if m else [])
    prov = [np.full(c.length, int(c.provenance), np.uint8) for c in chunks] + (
        [np.full(m, int(Provenance.FULL_PREFILL), np.uint8)] if m else [])
    return AssembledCache(
        chunk_ids=[c.chunk_id for c in chunks],
        chunk_lengths=lens,
        token_ids=parts(tok, np.int64),
        keys=keys,
        values=values,
        row_positions=parts(pos, np.int64),
        provenance=parts(prov, np.uint8),
        chunk_index=parts([np.full(n, i, np.int64) for i, n in enumerate(lens)], np.int64),
        local_index=parts([np.arange(n, dtype=np.int64) for n in lens], np.int64),
        prompt_length=m,
        model_fingerprint=fp,
    )


def assemble_decode_layout(chunks: Sequence[ChunkKV], rope_base: float, stream=None) -> AssembledCache:
    """``assemble`` and Kernel 1 in one pass: the chunks gathered in declared
    order with every key rotated from its stored position to its assembled
    (global) position while it is copied (``ifkv_assemble_gather_rotate``),
    i.e. ``to_decode_layout(assemble(chunks))`` with one read and one write
    of K instead of two of each.  Enqueued on ``stream`` (default: current)."""
    torch = _torch()
    if not chunks:
        raise ConfigurationError("nothing to assemble: no chunks")
    base = assemble_metadata(chunks)
    ref = chunks[0].keys
    L, _, Hkv, Dh = ref.shape
    n = base.context_length
    keys = torch.empty((L, n, Hkv, Dh), dtype=ref.dtype, device=ref.device)
    values = torch.empty_like(keys)
    starts = np.concatenate([[0], np.cumsum(base.chunk_lengths)[:-1]]).astype(np.int64)
    deltas = starts - np.array([int(c.prefill_positions[0]) for c in chunks], dtype=np.int64)
    uniq = sorted({int(d) for d in deltas if d != 0})
    cs_row = [uniq.index(int(d)) if d != 0 else -1 for d in deltas]
    # every chunk's stored positions must be one consecutive run (true for prefilled chunks)
    for c in chunks:
        if c.length and not np.array_equal(c.prefill_positions, c.prefill_positions[0] + np.arange(c.length)):
            raise ConfigurationError(f"chunk {c.chunk_id!r}: stored positions are not one run")
    cs = E.rope_table(np.asarray(uniq or [0], np.int64), Dh, rope_base, ref.device)
    if stream is not None:  # the gather may overlap later work of the current stream
        stream.wait_stream(torch.cuda.current_stream())
        for t in (cs, keys, values):  # used on the side stream: no reuse before its work is done
            t.record_stream(stream)
    with (torch.cuda.stream(stream) if stream is not None else _nullctx()):
        E.assemble_gather([c.keys for c in chunks], [c.values for c in chunks], keys, values, starts.tolist(),
                          cs_row=cs_row, cs=cs)
    base.keys, base.values = keys, values
    base.row_positions = np.concatenate([starts[i] + np.arange(c.length) for i, c in enumerate(chunks)])
    base.row_positions = base.row_positions.astype(np.int64)
    return base


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def assemble_metadata(chunks: Sequence[ChunkKV]) -> AssembledCache:
    """The host-side bookkeeping of ``assemble`` (checks, token ids, row
    positions, provenance, chunk mapping) with no device slab."""
    if not chunks:
        raise ConfigurationError("nothing to assemble: no chunks")
    fp = chunks[0].model_fingerprint
    ref = chunks[0].keys
    for c in chunks:
        if c.model_fingerprint != fp:
            raise ConfigurationError(f"chunk {c.chunk_id!r} was prefetched under a different model "
                                     f"(fingerprint {c.model_fingerprint:#x} != {fp:#x})")
        if c.n_layers != ref.shape[0] or c.keys.shape[2:] != ref.shape[2:] or c.keys.dtype != ref.dtype:
            raise ConfigurationError(f"chunk {c.chunk_id!r} KV shape mismatch")
    lens = [c.length for c in chunks]
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    return AssembledCache(
        chunk_ids=[c.chunk_id for c in chunks],
        chunk_lengths=lens,
        token_ids=cat([c.token_ids for c in chunks], np.int64),
        keys=None,
        values=None,
        row_positions=cat([c.prefill_positions for c in chunks], np.int64),
        provenance=cat([np.full(c.length, int(c.provenance), np.uint8) for c in chunks], np.uint8),
        chunk_index=cat([np.full(n, i, np.int64) for i, n in enumerate(lens)], np.int64),
        local_index=cat([np.arange(n, dtype=np.int64) for n in lens], np.int64),
        prompt_length=0,
        model_fingerprint=fp,
    )


def replace_entries(cache: AssembledCache, indices, new_kv, positions=None, inplace: bool = False) -> AssembledCache:
    """Overwrite exactly the listed context rows in every layer
    (cache.py:325-374).  new_kv: per-layer (k, v) row blocks [k, Hkv, Dh] or
    one (K, V) pair of [L, k, Hkv, Dh] tensors.  Out of place unless
    ``inplace``; untouched rows stay bit-identical."""
    torch = _torch()
    idx = np.asarray(indices, dtype=np.int64).ravel()
    n = cache.context_length
    if idx.size == 0:
        return cache
    if idx.min() < 0 or idx.max() >= n:
        raise ConfigurationError(f"replacement index outside context [0, {n})")
    if np.unique(idx).size != idx.size:
        raise ConfigurationError("duplicate replacement indices")
    if isinstance(new_kv, tuple) and len(new_kv) == 2 and hasattr(new_kv[0], "dim") and new_kv[0].dim() == 4:
        new_k, new_v = new_kv
    else:
        if len(new_kv) != cache.n_layers:
            raise ConfigurationError(f"new_kv has {len(new_kv)} layers, cache has {cache.n_layers}")
        new_k = torch.stack([torch.as_tensor(k) for k, _ in new_kv]).to(cache.keys.device, cache.keys.dtype)
        new_v = torch.stack([torch.as_tensor(v) for _, v in new_kv]).to(cache.keys.device, cache.keys.dtype)
    if new_k.shape[1] != idx.size or new_v.shape[1] != idx.size:
        raise ConfigurationError("replacement rows do not match indices")
    pos = idx.copy() if positions is None else np.asarray(positions, dtype=np.int64).ravel()
    if pos.size != idx.size:
        raise ConfigurationError("positions length does not match indices")
    keys = cache.keys if inplace else cache.keys.clone()
    values = cache.values if inplace else cache.values.clone()
    ti = torch.as_tensor(idx, device=keys.device)
    keys[:, ti] = new_k.to(keys.dtype)
    values[:, ti] = new_v.to(values.dtype)
    rp = cache.row_positions if inplace else cache.row_positions.copy()
    pv = cache.provenance if inplace else cache.provenance.copy()
    rp[idx] = pos
    pv[idx] = int(Provenance.RECOMPUTED_GLOBAL)
    return replace(cache, keys=keys, values=values, row_positions=rp, provenance=pv)


def decode_targets(cache: AssembledCache) -> np.ndarray:
    n = cache.context_length
    return np.concatenate([np.arange(n, dtype=np.int64), cache.row_positions[n:]])


def _delta_rows(deltas: np.ndarray):
    """Host half of the rotation table: per row, the index of its delta among
    the distinct nonzero deltas (-1 for delta 0), and those deltas."""
    deltas = np.asarray(deltas, dtype=np.int64)
    # runs of constant delta (one per chunk in the usual layouts): O(n), no sort
    cut = np.flatnonzero(np.diff(deltas)) + 1
    starts = np.concatenate([[0], cut])
    run_d = deltas[starts] if deltas.size else deltas
    if np.unique(run_d).size == run_d.size:  # every run has its own delta
        nz = run_d != 0
        rid = np.full(run_d.size, -1, np.int32)
        rid[nz] = np.arange(int(nz.sum()), dtype=np.int32)
        tab = np.repeat(rid, np.diff(np.concatenate([starts, [deltas.size]])))
        uniq_nz = run_d[nz]
    else:
        uniq, inv = np.unique(deltas, return_inverse=True)
        nzu = uniq != 0
        remap = np.full(uniq.size, -1, np.int32)
        remap[nzu] = np.arange(int(nzu.sum()), dtype=np.int32)
        tab = remap[inv.astype(np.int32)]
        uniq_nz = uniq[nzu]
    return tab.astype(np.int32), uniq_nz


def _delta_table(deltas: np.ndarray, d_head: int, rope_base: float, device):
    """Row table (int32, -1 for delta 0) and the fp64-derived cos/sin table
    of the distinct nonzero deltas."""
    tab, uniq_nz = _delta_rows(deltas)
    cs = E.rope_table(uniq_nz if uniq_nz.size else np.zeros(1, np.int64), d_head, rope_base, device)
    return E.h2d(tab, device), cs


def decode_view(cache: AssembledCache, rope_base: float):
    """(keys, values) with every row rotated to the global decode layout
    (cache.py:382-403).  Rows already there are copied bit-exactly.  Keys are
    a new tensor when any row moves, else the cache's own tensor."""
    torch = _torch()
    delta = decode_targets(cache) - cache.row_positions
    if not np.any(delta):
        return cache.keys, cache.values
    tab, cs = _delta_table(delta, cache.keys.shape[3], rope_base, cache.keys.device)
    out = torch.empty_like(cache.keys)
    E.rotate_rows(cache.keys, out, tab, cs)
    return out, cache.values


def to_decode_layout(cache: AssembledCache, rope_base: float, targets: Optional[np.ndarray] = None) -> AssembledCache:
    """Kernel 1 in place: rotate every context row to position = its index
    (the layout recompute and decoding run under) -- or, for a chunk shard,
    to its global index ``targets`` -- and update row_positions."""
    n = cache.context_length
    target = decode_targets(cache) if targets is None else np.concatenate(
        [np.asarray(targets, np.int64), cache.row_positions[n:]])
    delta = target - cache.row_positions
    if np.any(delta):
        tab, cs = _delta_table(delta, cache.keys.shape[3], rope_base, cache.keys.device)
        with E._Bracket("rotate_rows", int(np.count_nonzero(delta))):
            E.rotate_rows(cache.keys, cache.keys, tab, cs)
        cache.row_positions[:] = target
    return cache


def _fresh_prefill(weights, token_ids: np.ndarray):
    """Causal prefill of one token run at positions 0..n-1 through the shared
    layer stack (fresh K/V rows written in place, horizon = own index)."""
    torch = _torch()
    cfg = weights.config
    n = int(token_ids.size)
    if n > cfg.max_position:
        raise ConfigurationError(f"length {n} exceeds max_position {cfg.max_position}")
    if n and (token_ids.min() < 0 or token_ids.max() >= cfg.vocab_size):
        raise ConfigurationError("token id outside vocabulary")
    dev = weights.device
    keys = torch.empty((cfg.n_layers, n, cfg.kv_heads, cfg.d_head), dtype=weights.torch_dtype, device=dev)
    values = torch.empty_like(keys)
    ar = torch.arange(n, dtype=torch.int64, device=dev)
    ids = torch.as_tensor(token_ids, device=dev)
    E.layer_stack(weights, ids, ar, keys, values, ar, ar)
    return keys, values


def prefill_chunk(weights, chunk: ChunkSpec) -> ChunkKV:
    """Chunk-local prefill: positions 0..len-1, causal (cache.py:74-99)."""
    if chunk.local_length == 0:
        raise ConfigurationError(f"chunk {chunk.chunk_id!r} is empty")
    if chunk.local_length > weights.config.max_position:
        raise ConfigurationError(f"chunk {chunk.chunk_id!r} length {chunk.local_length} exceeds "
                                 f"max_position {weights.config.max_position}")
    keys, values = _fresh_prefill(weights, chunk.token_ids)
    return ChunkKV(chunk.chunk_id, chunk.token_ids.copy(), keys, values,
                   np.arange(chunk.local_length, dtype=np.int64), Provenance.PREFILLED_LOCAL, weights.fingerprint())


def prefill_chunks(weights, chunks: Sequence[ChunkSpec]) -> List[ChunkKV]:
    """Chunk-local prefill of many chunks in ONE pass (cache.py:74-99 for
    every chunk; the role of the reference's thread-pool prefill,
    costmodel.py:243-270): all tokens go through the layer stack together at
    their chunk-local positions under a block-diagonal causal mask (token i
    of a chunk attends rows chunk_start .. i), writing K/V straight into one
    store slab [L][sum len][Hkv][Dh].  The returned ChunkKVs are views of
    that store in the given order (each equals ``prefill_chunk`` of its chunk
    up to the accumulation order).  Batching turns K launches of M = len
    GEMMs into one launch per projection with M = sum len."""
    torch = _torch()
    cfg = weights.config
    if not chunks:
        return []
    for c in chunks:
        if c.local_length == 0:
            raise ConfigurationError(f"chunk {c.chunk_id!r} is empty")
        if c.local_length > cfg.max_position:
            raise ConfigurationError(f"chunk {c.chunk_id!r} length {c.local_length} exceeds "
                                     f"max_position {cfg.max_position}")
    lens = np.array([c.local_length for c in chunks], dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    n = int(lens.sum())
    tok = np.concatenate([np.asarray(c.token_ids, np.int64) for c in chunks])
    if tok.min() < 0 or tok.max() >= cfg.vocab_size:
        raise ConfigurationError("token id outside vocabulary")
    dev = weights.device
    store_k = torch.empty((cfg.n_layers, n, cfg.kv_heads, cfg.d_head), dtype=weights.torch_dtype, device=dev)
    store_v = torch.empty_like(store_k)
    local = np.concatenate([np.arange(m, dtype=np.int64) for m in lens])
    key_start = np.repeat(starts, lens)
    rows = torch.arange(n, dtype=torch.int64, device=dev)
    E.layer_stack(weights, E.h2d(tok, dev), E.h2d(local, dev), store_k, store_v, rows, rows,
                  key_start=E.h2d(key_start, dev))
    fp = weights.fingerprint()
    store = (store_k, store_v)
    return [ChunkKV(c.chunk_id, np.asarray(c.token_ids, np.int64).copy(), store_k[:, a:a + m], store_v[:, a:a + m],
                    np.arange(m, dtype=np.int64), Provenance.PREFILLED_LOCAL, fp, store=store, store_row0=a)
            for c, a, m in zip(chunks, starts.tolist(), lens.tolist())]


def full_prefill(weights, token_ids, chunk_id: str = "full") -> AssembledCache:
    """The whole context prefilled in one pass at global positions (cache.py:406-425)."""
    tok = np.asarray(token_ids, dtype=np.int64)
    if tok.size == 0:
        raise ConfigurationError("cannot prefill an empty context")
    keys, values = _fresh_prefill(weights, tok)
    ckv = ChunkKV(chunk_id, tok, keys, values, np.arange(tok.size, dtype=np.int64), Provenance.FULL_PREFILL,
                  weights.fingerprint())
    return assemble([ckv])


@dataclass(frozen=True)
class FidelityReport:
    frobenius: float
    max_abs: float


def cache_fidelity(cache: AssembledCache, reference: AssembledCache, rope_base: float) -> FidelityReport:
    """Distance between the decode views' context rows (cache.py:434-450)."""
    if cache.context_length != reference.context_length:
        raise ConfigurationError("caches cover different context lengths")
    if cache.n_layers != reference.n_layers:
        raise ConfigurationError("caches have different layer counts")
    n = cache.context_length
    ka, va = decode_view(cache, rope_base)
    kb, vb = decode_view(reference, rope_base)
    dk = (ka[:, :n].double() - kb[:, :n].double())
    dv = (va[:, :n].double() - vb[:, :n].double())
    fro = float((dk.square().sum() + dv.square().sum()).sqrt())
    worst = float(max(dk.abs().max(), dv.abs().max())) if n else 0.0
    return FidelityReport(frobenius=fro, max_abs=worst)


def chunk_from_host(chunk_id, token_ids, keys, values, positions, provenance, fingerprint, dtype, device="cuda"):
    """Upload host arrays (L, len, Hkv, Dh) as a ChunkKV."""
    torch = _torch()
    k = torch.as_tensor(np.ascontiguousarray(keys, dtype=np.float32)).to(device=device, dtype=dtype)
    v = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float32)).to(device=device, dtype=dtype)
    return ChunkKV(chunk_id, np.asarray(token_ids, np.int64), k, v, np.asarray(positions, np.int64),
                   Provenance(provenance), fingerprint)
