"""Chunk-sharding host logic on CPU: layout, horizon conversion, and the
cross-rank merges run over torch.distributed `gloo` with world size 2,
checked against unsharded oracle computations."""

import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2603_05353_b200 import sharding as SH


def test_zigzag_owners_balanced():
    own = SH.zigzag_owners(16, 4)
    assert own.tolist() == [0, 1, 2, 3, 3, 2, 1, 0] * 2
    for w in (1, 2, 3, 4, 8):
        own = SH.zigzag_owners(64, w)
        counts = np.bincount(own, minlength=w)
        assert counts.max() - counts.min() <= 2
        if 64 % (2 * w) == 0:
            # causal work (sum of chunk end positions) exactly balanced per 2R-chunk cycle
            work = np.bincount(own, weights=np.arange(64) + 1, minlength=w)
            assert work.max() == work.min()


def test_make_shard_rows_cover_context():
    lens = [5, 3, 7, 2, 4]
    shards = [SH.make_shard(lens, r, 2) for r in range(2)]
    allrows = np.sort(np.concatenate([s.global_rows for s in shards]))
    np.testing.assert_array_equal(allrows, np.arange(sum(lens)))
    for s in shards:
        assert np.all(np.diff(s.global_rows) > 0)


def test_local_horizon_is_visible_prefix():
    grows = torch.tensor([0, 1, 2, 7, 8, 12, 13, 14])
    hz = torch.tensor([0, 3, 7, 11, 14, 20])
    loc = torch.searchsorted(grows, hz, right=True) - 1
    for h, l in zip(hz.tolist(), loc.tolist()):
        assert l == int((grows <= h).sum()) - 1


def _worker(rank, world, store_path, fn, q):
    import torch.distributed as dist

    # a FileStore rendezvous: no TCP port to race for between test runs
    dist.init_process_group("gloo", init_method=f"file://{store_path}", rank=rank, world_size=world)
    try:
        q.put((rank, fn(SH.TorchComm())))
    except Exception as exc:  # pragma: no cover - surfaced in the parent
        q.put((rank, exc))
    finally:
        dist.destroy_process_group()


def _run_gloo(fn, world=2):
    import tempfile

    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as tmp:
        store = os.path.join(tmp, "store")
        procs = [ctx.Process(target=_worker, args=(r, world, store, fn, q)) for r in range(world)]
        for p in procs:
            p.start()
        out = dict(q.get(timeout=120) for _ in range(world))
        for p in procs:
            p.join(timeout=60)
    for v in out.values():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


# --- rank bodies (module level so spawn can pickle them) ----------------------


def _partial_state(q, k, v, horizon):
    """Softmax state (normalised ctx, max, sum) of q over a key subset; rows
    that see no key give (0, -inf, 0).  q [S,H,Dh], k/v [n,H,Dh] (MHA)."""
    S, H, Dh = q.shape
    logits = torch.einsum("shd,nhd->shn", q, k) / np.sqrt(Dh)
    n = k.shape[0]
    mask = torch.arange(n)[None, None, :] <= horizon[:, None, None]
    logits = torch.where(mask, logits, torch.tensor(float("-inf"), dtype=logits.dtype))
    m = logits.max(-1).values
    safe = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    e = torch.exp(logits - safe[..., None]) * mask
    l = e.sum(-1)
    ctx = torch.einsum("shn,nhd->shd", e, v) / torch.where(l > 0, l, torch.ones_like(l))[..., None]
    return ctx, torch.stack([torch.where(l > 0, m, torch.full_like(m, float("-inf"))), l], -1)


def _body_query_merge(comm):
    torch.manual_seed(0)
    S, H, Dh, lens = 40, 4, 16, [30, 20, 25, 15, 10]
    N = sum(lens)
    q, k, v = torch.randn(S, H, Dh, dtype=torch.float64), torch.randn(N, H, Dh, dtype=torch.float64), \
        torch.randn(N, H, Dh, dtype=torch.float64)
    hz = torch.sort(torch.randperm(N)[:S]).values
    shard = SH.make_shard(lens, comm.rank, comm.world)
    grows = torch.as_tensor(shard.global_rows)
    loc_hz = torch.searchsorted(grows, hz, right=True) - 1
    ctx, ml = _partial_state(q, k[grows], v[grows], loc_hz)
    merged = SH.merge_query_states(comm.all_gather(ctx), comm.all_gather(ml))
    full, _ = O.prefix_attention(q.numpy(), k.numpy(), v.numpy(), hz.numpy())
    return float(np.max(np.abs(merged.numpy() - full)))


def _body_prompt_merge(comm):
    torch.manual_seed(1)
    G, M, H, Dh, lens = 1, 6, 2, 8, [9, 7, 11, 5]
    N = sum(lens)
    q = torch.randn(M, H, Dh, dtype=torch.float64)
    k, v = torch.randn(N + M, H, Dh, dtype=torch.float64), torch.randn(N + M, H, Dh, dtype=torch.float64)
    shard = SH.make_shard(lens, comm.rank, comm.world)
    grows = torch.as_tensor(shard.global_rows)
    # context keys: all visible; prompt keys (causal) counted on rank 0 only
    kk, vv = k[grows], v[grows]
    hz = torch.full((M,), len(grows) - 1)
    if comm.rank == 0:
        kk, vv = torch.cat([kk, k[N:]]), torch.cat([vv, v[N:]])
        hz = len(grows) + torch.arange(M)
    ctx, ml = _partial_state(q, kk, vv, hz)  # [M, H, Dh], [M, H, 2]
    ctx_g, ml_g = ctx[None], ml.permute(1, 0, 2)[None]  # [G, M, H, Dh], [G, H, M, 2]
    merged, mlm = SH.merge_prompt_states(comm.all_gather(ctx_g), comm.all_gather(ml_g))
    full, probs = O.prefix_attention(q.numpy(), k.numpy(), v.numpy(), N + np.arange(M), want_probs=True)
    return float(np.max(np.abs(merged[0].numpy() - full)))


def _body_topk(comm):
    rng = np.random.default_rng(3)
    N, k = 500, 77
    s = rng.choice([0.1, 0.2, 0.3, 0.35], size=N).astype(np.float32)
    shard = SH.make_shard([100] * 5, comm.rank, comm.world)
    loc = torch.as_tensor(s[shard.global_rows])
    kl = min(k, loc.numel())
    order = sorted(range(loc.numel()), key=lambda i: (-float(loc[i]), int(shard.global_rows[i])))[:kl]
    cand_s = loc[order]
    cand_i = torch.as_tensor(shard.global_rows[order])
    got = SH.merge_topk(comm.all_gather_var(cand_s), comm.all_gather_var(cand_i), k)
    want = O.select_topk(s.astype(np.float64), k)
    return bool(np.array_equal(got.numpy(), want))


def test_gloo_query_state_merge_matches_full_attention():
    errs = _run_gloo(_body_query_merge)
    assert max(errs) < 1e-12


def test_gloo_prompt_state_merge_matches_full_attention():
    errs = _run_gloo(_body_prompt_merge)
    assert max(errs) < 1e-12


def test_gloo_topk_candidate_merge_exact():
    assert all(_run_gloo(_body_topk))


def _body_all_to_all(comm):
    """Uneven (and empty) per-destination parts: rank r sends r + d rows to d,
    every row tagged (source, destination, index)."""
    parts = [torch.tensor([[comm.rank, d, i] for i in range(comm.rank + d)], dtype=torch.int64).reshape(-1, 3)
             for d in range(comm.world)]
    got = comm.all_to_all(parts)
    ok = len(got) == comm.world
    for src, t in enumerate(got):
        want = torch.tensor([[src, comm.rank, i] for i in range(src + comm.rank)], dtype=torch.int64).reshape(-1, 3)
        ok = ok and torch.equal(t, want)
    return ok


def test_gloo_all_to_all_uneven_and_empty():
    assert all(_run_gloo(_body_all_to_all))
