"""Chunk-sharded query-time context assembly across the GPUs of one box
(the reference has no distributed path -- its cost model
`costmodel.py:127-177` describes the "communicate only the selected tokens"
scheme this implements).

Layout: chunk c lives on rank ``zigzag_owners(K, R)[c]`` (zig-zag over 2R
slots so every rank holds early and late chunks and the causal work is
balanced).  Each rank keeps only its chunks' KV (its own assembled slab,
local rows in ascending global order) and a replica of the weights.

Scoring (selection.py:127-183): every rank runs the prompt forward against
its own chunks; after every layer the per-rank softmax states (normalised
context, max, sum) are all-gathered and merged in rank order (identical on
every rank, deterministic); the prompt's own keys are counted once (rank 0).
At the capture layer each rank scores its own rows with the merged (max, sum)
and takes a local top-k; the (score, global index) candidates are
all-gathered and merged with the reference's tie rule -- exact, because the
global top-k is contained in the union of the local top-k's.

Recompute (recompute.py:67-122): every rank advances the selected tokens it
owns through the layer stack (weights replicated, owner-computes) and
scatters their K/V into its slab; per layer the selected queries are
all-gathered, every rank computes partial causal attention of all of them
against its local keys (``ifkv_recompute_attn_partial``), and the partials
are sent back to the owners (all-to-all) and merged in rank order.  Traffic
per layer is O(k), not ring attention's O(N).

``TorchComm`` runs the collectives over torch.distributed (NCCL on GPUs, gloo
on CPU tensors); ``ThreadComm`` runs R ranks as threads of one process on one
device so the sharded data path is exercised on a single GPU.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import engine as E
from .cache import AssembledCache, Provenance, to_decode_layout
from .errors import ConfigurationError
from .selection import SelectionConfig, SelectionResult, default_norm_layer


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------


class Comm:
    """Single-rank communicator (collectives are identities)."""

    world = 1
    rank = 0

    def all_gather(self, t) -> list:
        return [t]

    def all_gather_var(self, t, sizes=None) -> list:
        """all_gather for tensors whose first dimension differs per rank
        (``sizes``: the per-rank first dimensions when already known)."""
        return self.all_gather(t)

    def all_to_all(self, parts: list, recv_sizes=None) -> list:
        return list(parts)

    def all_gather_var_async(self, t, sizes):
        """Start all_gather_var; ``.wait()`` on the handle returns the list.
        Lets the caller compute on its own data while the gather is in flight."""
        return _Done(self.all_gather_var(t, sizes))


class _Done:
    def __init__(self, value):
        self.value = value

    def wait(self):
        return self.value


class _Pending:
    def __init__(self, work, bufs, sizes, keep):
        self.work, self.bufs, self.sizes, self.keep = work, bufs, sizes, keep

    def wait(self):
        self.work.wait()  # NCCL: the current stream waits for the collective's stream
        return [x[:n] for x, n in zip(self.bufs, self.sizes)]


class TorchComm(Comm):
    """torch.distributed collectives (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, t):
        t = t.contiguous()
        out = [t.new_empty(t.shape) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return out

    def _sizes(self, n: int, device):
        torch = _torch()
        s = torch.tensor([n], dtype=torch.int64, device=device)
        return [int(x.item()) for x in self.all_gather(s)]

    def all_gather_var(self, t, sizes=None):
        t = t.contiguous()
        if sizes is None:  # one host round trip; callers in per-layer loops pass known sizes
            sizes = self._sizes(t.shape[0], t.device)
        cap = max(sizes) if sizes else 0
        pad = t.new_zeros((cap,) + tuple(t.shape[1:]))
        pad[: t.shape[0]] = t
        return [x[:n] for x, n in zip(self.all_gather(pad), sizes)]

    def all_gather_var_async(self, t, sizes):
        t = t.contiguous()
        cap = max(sizes) if sizes else 0
        pad = t.new_zeros((cap,) + tuple(t.shape[1:]))
        pad[: t.shape[0]] = t
        bufs = [pad.new_empty(pad.shape) for _ in range(self.world)]
        work = self.dist.all_gather(bufs, pad, group=self.group, async_op=True)
        return _Pending(work, bufs, sizes, pad)

    def all_to_all(self, parts, recv_sizes=None):
        parts = [p.contiguous() for p in parts]
        torch = _torch()
        if self.dist.get_backend(self.group) == "gloo":
            # gloo has no alltoall: all-gather every rank's concatenated parts
            # (and their sizes) and keep the slices addressed to this rank
            sizes = torch.tensor([p.shape[0] for p in parts], dtype=torch.int64, device=parts[0].device)
            all_sizes = [s.tolist() for s in self.all_gather(sizes)]
            all_flat = self.all_gather_var(torch.cat(parts), [sum(x) for x in all_sizes])
            out = []
            for r in range(self.world):
                off = sum(all_sizes[r][: self.rank])
                out.append(all_flat[r][off: off + all_sizes[r][self.rank]])
            return out
        if recv_sizes is None:  # receive sizes first (first dimension may differ)
            send_n = torch.tensor([p.shape[0] for p in parts], dtype=torch.int64, device=parts[0].device)
            recv_n = torch.empty_like(send_n)
            self.dist.all_to_all_single(recv_n, send_n, group=self.group)
            recv_sizes = recv_n.tolist()
        recv = [parts[0].new_empty((int(n),) + tuple(parts[0].shape[1:])) for n in recv_sizes]
        self.dist.all_to_all(recv, parts, group=self.group)
        return recv


class ThreadComm(Comm):
    """R ranks as threads of one process sharing one device (collectives are
    list exchanges behind a barrier).  Used to run the sharded data path,
    kernels included, on a single GPU."""

    def __init__(self, world: int, rank: int, shared: dict):
        self.world, self.rank, self.shared = world, rank, shared

    @staticmethod
    def run(world: int, fn: Callable[["ThreadComm"], object]) -> list:
        shared = {"slots": [None] * world, "barrier": threading.Barrier(world)}
        results, errors = [None] * world, [None] * world

        def body(r):
            try:
                results[r] = fn(ThreadComm(world, r, shared))
            except BaseException as exc:  # noqa: BLE001 -- re-raised below
                errors[r] = exc
                shared["barrier"].abort()

        threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for e in errors:
            if e is not None and not isinstance(e, threading.BrokenBarrierError):
                raise e
        for e in errors:
            if e is not None:
                raise e
        return results

    def _exchange(self, value, pick):
        """Publish `value`, read the others' through `pick` (which copies), and
        only then release the writers: every copy is enqueued on the shared
        stream before any rank can enqueue a write to its published tensors."""
        slots, bar = self.shared["slots"], self.shared["barrier"]
        slots[self.rank] = value
        bar.wait()
        out = [pick(r, slots[r]) for r in range(self.world)]
        bar.wait()
        return out

    def all_gather(self, t):
        return self._exchange(t, lambda r, x: x if r == self.rank else x.clone())

    def all_gather_var(self, t, sizes=None):
        return self.all_gather(t)

    def all_to_all(self, parts, recv_sizes=None):
        return self._exchange(list(parts), lambda r, x: x[self.rank].clone())


# ---------------------------------------------------------------------------
# layout
# ---------------------------------------------------------------------------


def zigzag_owners(n_chunks: int, world: int) -> np.ndarray:
    """Chunk c -> rank: slot c mod 2R, folded (r, 2R-1-r) so each rank gets
    one early and one late chunk per 2R chunks (balanced causal work)."""
    slot = np.arange(n_chunks) % (2 * world)
    return np.where(slot < world, slot, 2 * world - 1 - slot).astype(np.int64)


@dataclass
class Shard:
    rank: int
    world: int
    chunk_ids: List[int]  # global declared-order indices of the owned chunks (ascending)
    global_rows: np.ndarray  # global context index of every local row (ascending)
    n_context: int
    rank_rows: Optional[List[int]] = None  # context rows held by every rank (known to all ranks)
    row_owner: Optional[np.ndarray] = None  # rank holding every global context row


def make_shard(chunk_lengths: Sequence[int], rank: int, world: int, owners: Optional[np.ndarray] = None) -> Shard:
    lens = np.asarray(chunk_lengths, np.int64)
    owners = zigzag_owners(len(lens), world) if owners is None else np.asarray(owners)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    mine = [int(c) for c in np.flatnonzero(owners == rank)]
    rows = [starts[c] + np.arange(lens[c]) for c in mine]
    rank_rows = [int(lens[owners == r].sum()) for r in range(world)]
    return Shard(rank, world, mine, np.concatenate(rows).astype(np.int64) if rows else np.zeros(0, np.int64),
                 int(lens.sum()), rank_rows, np.repeat(owners, lens).astype(np.int64))


# ---------------------------------------------------------------------------
# merges (fixed rank order -> identical, deterministic results on every rank)
# ---------------------------------------------------------------------------


def merge_softmax_states(ctxs: Sequence, mls: Sequence, head_axis_ml: bool = True):
    """Merge per-rank softmax states.  ctx_r: normalised context (any float
    dtype), ml_r: (max, sum) in the last dim, broadcast-compatible with ctx_r
    after unsqueezing the feature dim.  Returns (ctx fp32, ml)."""
    torch = _torch()
    m = torch.stack([x[..., 0] for x in mls])  # [R, ...]
    l = torch.stack([x[..., 1] for x in mls])
    mx = torch.max(m, dim=0).values
    safe = torch.where(torch.isfinite(mx), mx, torch.zeros_like(mx))
    w = torch.where(l > 0, l * torch.exp(m - safe), torch.zeros_like(l))  # [R, ...]
    lt = w.sum(0)
    return w, mx, lt


def merge_prompt_states(ctxs: Sequence, mls: Sequence):
    """ctx_r [G, M, H, Dh] fp32, ml_r [G, H, M, 2] -> merged (ctx, ml)."""
    torch = _torch()
    w, mx, lt = merge_softmax_states(ctxs, mls)
    acc = torch.zeros_like(ctxs[0])
    for r, c in enumerate(ctxs):
        acc += c * w[r].transpose(1, 2).unsqueeze(-1)  # [G, H, M] -> [G, M, H, 1]
    ctx = acc / torch.where(lt > 0, lt, torch.ones_like(lt)).transpose(1, 2).unsqueeze(-1)
    return ctx, torch.stack([mx, lt], dim=-1)


def merge_query_states(ctxs: Sequence, mls: Sequence):
    """ctx_r [S, H, Dh], ml_r [S, H, 2] -> merged normalised ctx [S, H, Dh]
    (fp32, or fp64 for fp64 inputs)."""
    torch = _torch()
    w, _, lt = merge_softmax_states(ctxs, mls)
    dt = torch.float64 if ctxs[0].dtype == torch.float64 else torch.float32
    acc = torch.zeros(ctxs[0].shape, dtype=dt, device=ctxs[0].device)
    for r, c in enumerate(ctxs):
        acc += c.to(dt) * w[r].to(dt).unsqueeze(-1)
    return acc / torch.where(lt > 0, lt, torch.ones_like(lt)).unsqueeze(-1)


def merge_topk(scores: Sequence, indices: Sequence, k: int):
    """Global top-k of per-rank candidates by (score desc, global index asc),
    returned ascending -- the reference's rule (selection.py:172-183)."""
    torch = _torch()
    s = torch.cat([x.float().reshape(-1) for x in scores])
    i = torch.cat([x.reshape(-1) for x in indices]).to(torch.int64)
    if k > s.numel():
        raise ConfigurationError(f"k ({k}) exceeds candidate count ({s.numel()})")
    b = s.view(torch.int32).to(torch.int64)
    b = torch.where(s == 0, torch.zeros_like(b), b)  # -0 == +0
    key = torch.where(b < 0, -(b & 0x7FFFFFFF) - 1, b)  # order-preserving int for float bits
    # sort by score desc, then index asc (stable sort on index first)
    o = torch.argsort(i, stable=True)
    o = o[torch.argsort(key[o], descending=True, stable=True)]
    return torch.sort(i[o[:k]]).values


# ---------------------------------------------------------------------------
# sharded path
# ---------------------------------------------------------------------------


def sharded_select(weights, shard: Shard, cache: AssembledCache, prompt_token_ids, config: SelectionConfig,
                   comm: Comm) -> SelectionResult:
    """Attention-norm selection (GLOBAL geometry) over chunk shards.  Returns
    the global selected set (identical on every rank) and this rank's scores
    for its local rows."""
    torch = _torch()
    cfg = weights.config
    from .positions import GeometryConfig, GeometryMode
    from .selection import Strategy

    if config.strategy != Strategy.ATTENTION_NORM:
        raise ConfigurationError(f"sharded selection implements the attention-norm strategy only, got "
                                 f"{config.strategy.value!r}")
    if config.score_precision != "fp32":
        raise ConfigurationError("sharded selection scores in the fp32-accurate mode only (score_precision='fp32')")
    geo = config.geometry
    mode = geo.mode if isinstance(geo, GeometryConfig) else (GeometryMode.parse(geo) if geo is not None else None)
    if mode not in (None, GeometryMode.GLOBAL):
        raise ConfigurationError(f"sharded selection scores under GLOBAL geometry only, got {mode.value!r}")
    prompt = np.asarray(prompt_token_ids, np.int64)
    n_local = cache.context_length
    if n_local != shard.global_rows.size:
        raise ConfigurationError("shard cache does not match the shard layout")
    nl = config.norm_layer if config.norm_layer is not None else default_norm_layer(cfg.n_layers)
    N = shard.n_context
    prompt_pos = N + np.arange(prompt.size, dtype=np.int64)
    group = E.PromptGroup(prompt, prompt_pos, E.segments_from_deltas(shard.global_rows - cache.row_positions[:n_local]))

    def hook(ctx, ml):
        if comm.world == 1:
            return ctx, ml
        if ctx.is_cuda and ctx.dtype == torch.float32:  # one fused merge kernel per layer
            return E.merge_prompt_states(torch.stack(comm.all_gather(ctx)), torch.stack(comm.all_gather(ml)))
        return merge_prompt_states(comm.all_gather(ctx), comm.all_gather(ml))

    out = E.prompt_forward(weights, cache.keys, cache.values, [group], capture_layer=nl, merge_hook=hook,
                           include_prompt=shard.rank == 0)
    scores = out.scores[:n_local]
    k = config.resolve_budget(N)
    kl = min(k, n_local)
    if kl:
        from .selection import select_topk

        loc = select_topk(scores, kl)
    else:
        loc = torch.zeros(0, dtype=torch.int64, device=scores.device)
    grows = torch.as_tensor(shard.global_rows, device=scores.device)
    cand_idx = grows.index_select(0, loc)
    cand_s = scores.index_select(0, loc)
    # every rank's candidate count is known from the layout: no host round trip
    sizes = [min(k, n) for n in shard.rank_rows] if shard.rank_rows is not None else None
    sel = merge_topk(comm.all_gather_var(cand_s, sizes), comm.all_gather_var(cand_idx, sizes), k)
    return SelectionResult(scores=scores, selected=sel, strategy="attention-norm", geometry="GLOBAL")


def sharded_reorder(weights, chunks: Sequence, chunk_kvs: Sequence, shard: Shard, prompt_token_ids, budget: int,
                    comm: Comm, norm_layer: Optional[int] = None, chunk_score: str = "sum"):
    """Information-flow reordering over chunk shards (reorder.py:57-181, SURVEY
    §8e item 4).  The first pass is per chunk and needs no exchange: each rank
    scores its own chunks (``chunk_kvs``: this rank's KVs, in ``shard.chunk_ids``
    order); the importances are all-gathered and every rank computes the same
    stable permutation.  Chunks stay on their ranks: the permuted layout only
    changes their global rows.  Returns (permutation, importances, the shard in
    the permuted layout, this rank's cache assembled in that layout's order)."""
    torch = _torch()
    from .cache import assemble
    from .reorder import score_chunks

    n_total = sum(c.local_length for c in chunks)
    mine = [chunks[c] for c in shard.chunk_ids]
    if mine:
        imp_local, _ = score_chunks(weights, mine, prompt_token_ids, budget, norm_layer=norm_layer,
                                    chunk_score=chunk_score, prefilled=list(chunk_kvs),
                                    _context=(len(chunks), n_total))
    else:
        imp_local = np.zeros(0, np.float64)
    dev = weights.device
    csizes = None
    if shard.row_owner is not None:  # chunks per rank, known from the layout
        starts0 = np.concatenate([[0], np.cumsum([c.local_length for c in chunks])[:-1]]).astype(np.int64)
        csizes = np.bincount(shard.row_owner[starts0], minlength=shard.world).tolist()
    ids = comm.all_gather_var(torch.as_tensor(np.asarray(shard.chunk_ids, np.int64), device=dev), csizes)
    imps = comm.all_gather_var(torch.as_tensor(np.asarray(imp_local, np.float64), device=dev), csizes)
    importances = np.zeros(len(chunks), np.float64)
    for i, v in zip(ids, imps):
        importances[i.cpu().numpy()] = v.cpu().numpy()
    permutation = np.argsort(importances, kind="stable").astype(np.int64)  # most important last
    lens = np.asarray([c.local_length for c in chunks], np.int64)
    slot_of = np.empty(len(chunks), np.int64)
    slot_of[permutation] = np.arange(len(chunks))
    starts = np.concatenate([[0], np.cumsum(lens[permutation])[:-1]])  # global start of each slot
    order = sorted(range(len(shard.chunk_ids)), key=lambda i: slot_of[shard.chunk_ids[i]])
    owned = [shard.chunk_ids[i] for i in order]  # ascending in the permuted layout
    rows = [starts[slot_of[c]] + np.arange(lens[c]) for c in owned]
    owners_perm = np.empty(int(n_total), np.int64)  # rank of every row in the permuted layout
    all_owners = shard.row_owner
    if all_owners is not None:
        chunk_owner = np.array([all_owners[int(np.sum(lens[:c]))] for c in range(len(chunks))], np.int64)
        for c in range(len(chunks)):
            owners_perm[starts[slot_of[c]]: starts[slot_of[c]] + lens[c]] = chunk_owner[c]
    pshard = Shard(shard.rank, shard.world, owned,
                   np.concatenate(rows).astype(np.int64) if rows else np.zeros(0, np.int64), int(n_total),
                   shard.rank_rows, owners_perm if all_owners is not None else None)
    local = assemble([chunk_kvs[i] for i in order])
    return permutation, importances, pshard, local


def sharded_recompute(weights, shard: Shard, cache: AssembledCache, selected_global, comm: Comm) -> AssembledCache:
    """Recompute the globally selected tokens, each on the rank owning it,
    with attention over every rank's keys; K/V scattered into the owners'
    slabs in place.  Every rank must call this (collectives per layer)."""
    torch = _torch()
    cfg = weights.config
    dev = cache.keys.device
    H, Hkv, Dh = cfg.n_heads, cfg.kv_heads, cfg.d_head
    grows_np = shard.global_rows
    grows = torch.as_tensor(grows_np, device=dev)
    sel = torch.as_tensor(selected_global, device=dev).to(torch.int64)
    pos = torch.searchsorted(grows, sel)
    mine = (pos < grows.numel()) & (grows.index_select(0, pos.clamp(max=max(grows.numel() - 1, 0))) == sel) \
        if grows.numel() else torch.zeros_like(sel, dtype=torch.bool)
    sel_g = sel[mine]  # global indices of my selected tokens (ascending)
    dst = pos[mine]  # their local slab rows
    to_decode_layout(cache, cfg.rope_base, targets=grows_np)
    ids = cache.token_ids_device().index_select(0, dst)

    # per-rank query counts and the local causal horizons of every rank's
    # queries are layer-invariant: exchange them once, so the per-layer
    # collectives below need no host round trip (the GPU never drains)
    if shard.row_owner is not None:  # per-rank query counts from the (replicated) selected set: one host sync
        owner = torch.as_tensor(shard.row_owner, device=dev)
        sizes = torch.bincount(owner.index_select(0, sel), minlength=comm.world).tolist()
    else:
        sizes = None
    hz_parts = comm.all_gather_var(sel_g, sizes)
    sizes = [int(h.numel()) for h in hz_parts]
    hz_loc = [torch.searchsorted(grows, hp, right=True) - 1 for hp in hz_parts]  # local causal horizons
    hz_mine = hz_loc[comm.rank]
    others = [r for r in range(comm.world) if r != comm.rank]
    hz_rem = torch.cat([hz_loc[r] for r in others]) if others else hz_mine[:0]
    mine_n = [sizes[comm.rank]] * comm.world

    def attn_fn(li, q_local, k_layer, v_layer):
        # this rank's queries against its keys while the other ranks' queries
        # are gathered (NCCL runs the gather on its own stream), then theirs
        pending = comm.all_gather_var_async(q_local, sizes)
        ctx_l, ml_l = E.recompute_attn_partial(q_local, k_layer, v_layer, hz_mine, H, Hkv, Dh)
        if comm.world == 1:  # one shard: the partial is the whole attention
            return ctx_l
        parts = pending.wait()
        q_rem = torch.cat([parts[r] for r in others])
        ctx_r, ml_r = E.recompute_attn_partial(q_rem, k_layer, v_layer, hz_rem, H, Hkv, Dh)
        send_ctx, send_ml, off = [], [], 0
        for r in range(comm.world):
            if r == comm.rank:
                send_ctx.append(ctx_l)
                send_ml.append(ml_l)
            else:
                send_ctx.append(ctx_r[off: off + sizes[r]])
                send_ml.append(ml_r[off: off + sizes[r]])
                off += sizes[r]
        back_ctx = comm.all_to_all(send_ctx, mine_n)
        back_ml = comm.all_to_all(send_ml, mine_n)
        if q_local.dtype == torch.bfloat16:  # one fused merge kernel instead of ~10 elementwise passes
            return E.merge_partials(torch.stack(back_ctx), torch.stack(back_ml))
        return merge_query_states(back_ctx, back_ml).to(q_local.dtype)

    E.layer_stack(weights, ids, sel_g, cache.keys, cache.values, dst, sel_g, attn_fn=attn_fn)
    d = dst.cpu().numpy()
    cache.row_positions[d] = sel_g.cpu().numpy()
    cache.provenance[d] = int(Provenance.RECOMPUTED_GLOBAL)
    return cache
