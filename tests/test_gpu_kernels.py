"""Kernel-level parity on the GPU: each C-ABI entry point against the oracle
(or an exact NumPy statement of the same arithmetic) on seeded inputs."""

import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def test_rope_table_fp64_angles(T, cuda):
    from paper_2603_05353_b200 import engine as E

    pos = np.array([0, 1, 7, 4095, 32767, 131071, -5, -2048], dtype=np.int64)
    for dh, base in ((128, 500000.0), (8, 10000.0), (128, 1e6)):
        cs = E.rope_table(pos, dh, base, cuda).cpu().numpy()
        ang = pos[:, None].astype(np.float64) * O.rope_theta(dh, base)[None, :]
        np.testing.assert_allclose(cs[..., 0], np.cos(ang).astype(np.float32), atol=2e-7)
        np.testing.assert_allclose(cs[..., 1], np.sin(ang).astype(np.float32), atol=2e-7)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("in_place", [True, False])
def test_rotate_rows_kernel1(T, cuda, dtype, in_place):
    from paper_2603_05353_b200 import cache as C
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(0)
    L, n, hkv, dh = 3, 777, 8, 128
    tdt = T.bfloat16 if dtype == "bf16" else T.float32
    x = T.as_tensor(rng.standard_normal((L, n, hkv, dh)), dtype=T.float32).to(cuda, tdt)
    deltas = rng.integers(-3000, 40000, n)
    deltas[::5] = 0
    tab, cs = C._delta_table(deltas, dh, 500000.0, cuda)
    src = x.clone()
    out = src if in_place else T.empty_like(src)
    E.rotate_rows(src, out, tab, cs)
    xs = x.double().cpu().numpy()
    want = np.stack([O.rope_rotate(xs[l], deltas, 500000.0) for l in range(L)])
    got = out.double().cpu().numpy()
    tol = 8e-3 if dtype == "bf16" else 2e-6
    assert np.max(np.abs(got - want)) <= tol * np.max(np.abs(want))
    zero = deltas == 0
    assert np.array_equal(got[:, zero], xs[:, zero])  # delta 0 rows bit-exact


def test_assemble_gather_bitwise(T, cuda):
    from paper_2603_05353_b200 import cache as C

    rng = np.random.default_rng(1)
    L, hkv, dh = 2, 4, 128
    lens = [256, 100, 3, 300]
    chunks = []
    for i, n in enumerate(lens):
        k = rng.standard_normal((L, n, hkv, dh))
        v = rng.standard_normal((L, n, hkv, dh))
        chunks.append(C.chunk_from_host(f"c{i}", np.arange(n) % 50, k, v, np.arange(n), 0, 123, T.bfloat16))
    cache = C.assemble(chunks)
    want_k = T.cat([c.keys for c in chunks], dim=1)
    want_v = T.cat([c.values for c in chunks], dim=1)
    assert T.equal(cache.keys, want_k) and T.equal(cache.values, want_v)
    assert cache.mapping(256) == ("c1", 0) and cache.mapping(358) == ("c2", 2) and cache.mapping(359) == ("c3", 0)
    perm = C.assemble([chunks[2], chunks[0]])
    assert T.equal(perm.keys, T.cat([chunks[2].keys, chunks[0].keys], dim=1))


def _brute_topk(s, k):
    return np.sort(np.lexsort((np.arange(s.size), -s))[:k])


@pytest.mark.parametrize("n,k", [(1, 0), (1, 1), (10, 3), (2048, 308), (32768, 4916), (131072, 19661),
                                 (5000, 5000), (4097, 1)])
def test_topk_exact_with_ties(T, cuda, n, k):
    from paper_2603_05353_b200.selection import select_topk

    rng = np.random.default_rng(n + k)
    for trial in range(3):
        if trial == 0:
            s = rng.random(n).astype(np.float32)
        elif trial == 1:
            s = rng.choice(np.array([0.1, 0.25, 0.5, 0.77], np.float32), size=n)
        else:
            s = (rng.random(n) * 1e-3 + 1.0).astype(np.float32)
            s[rng.integers(0, n, max(1, n // 10))] = 0.0
        got = select_topk(T.as_tensor(s, device=cuda), k).cpu().numpy()
        np.testing.assert_array_equal(got, _brute_topk(s.astype(np.float64), k))


def test_topk_segments_aggregate(T, cuda):
    from paper_2603_05353_b200 import _native as N
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(5)
    lens = [256, 2048, 7, 1, 300]
    s = rng.random(sum(lens)).astype(np.float32)
    s[260:270] = 0.5
    begin = np.concatenate([[0], np.cumsum(lens)])
    ks = [39, 308, 7, 1, 0]
    for mode in ("sum", "mean", "max"):
        idx, agg, ob = E.topk_segments(T.as_tensor(s, device=cuda), begin, ks, N.AGG_CODES[mode])
        idx, agg = idx.cpu().numpy(), agg.cpu().numpy()
        for i in range(len(lens)):
            seg = s[begin[i]:begin[i + 1]].astype(np.float64)
            want = _brute_topk(seg, ks[i])
            np.testing.assert_array_equal(idx[ob[i]:ob[i + 1]] - begin[i], want)
            assert agg[i] == pytest.approx(O.aggregate(seg[want], mode), rel=1e-12, abs=0)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("hkv,dh", [(8, 128), (4, 128), (2, 16), (1, 8)])
def test_recompute_attention_kernel(T, cuda, dtype, hkv, dh):
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(hkv * dh)
    H = 4 * hkv if hkv > 1 else 2
    n = 1500
    sel = np.sort(rng.choice(n, 300, replace=False))
    tdt = T.bfloat16 if dtype == "bf16" else T.float32
    q = T.as_tensor(rng.standard_normal((sel.size, H, dh)), dtype=T.float32).to(cuda, tdt)
    k = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, tdt)
    v = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, tdt)
    out = E.recompute_attn(q, k, v, T.as_tensor(sel, device=cuda), H, hkv, dh)
    want, _ = O.prefix_attention(q.double().cpu().numpy(), k.double().cpu().numpy(), v.double().cpu().numpy(), sel)
    got = out.double().cpu().numpy()
    tol = 1e-2 if dtype == "bf16" else 1e-5
    assert np.max(np.abs(got - want)) <= tol * np.max(np.abs(want))


@pytest.mark.parametrize("G", [1, 2, 4, 7, 8])
def test_recompute_attention_tcgen05_vs_simt(T, cuda, G):
    """The tcgen05 kernel against the SIMT fp32-softmax kernel (and the oracle)
    on a multi-block causal span: 4096 keys, 700 selected rows."""
    from paper_2603_05353_b200 import _native as N
    from paper_2603_05353_b200 import engine as E

    assert N.call("ifkv_recompute_attn_tc_supported", N.IFKV_BF16, 4 * G, 4, 128) == 1
    rng = np.random.default_rng(G)
    hkv, dh, n = 4, 128, 4096
    H = hkv * G
    sel = np.sort(rng.choice(n, 700, replace=False))
    q = T.as_tensor(rng.standard_normal((sel.size, H, dh)) * 2, dtype=T.float32).to(cuda, T.bfloat16)
    k = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    v = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    hz = T.as_tensor(sel, device=cuda)
    tc = E.recompute_attn(q, k, v, hz, H, hkv, dh).double().cpu().numpy()
    simt = E.recompute_attn(q, k, v, hz, H, hkv, dh, impl="simt").double().cpu().numpy()
    want, _ = O.prefix_attention(q.double().cpu().numpy(), k.double().cpu().numpy(), v.double().cpu().numpy(), sel)
    scale = np.max(np.abs(want))
    assert np.max(np.abs(simt - want)) <= 1e-2 * scale
    assert np.max(np.abs(tc - want)) <= 1e-2 * scale


@pytest.mark.parametrize("partial,n_empty", [(False, 0), (True, 7), (True, 130)])
def test_recompute_attention_unsorted_and_empty_horizons(T, cuda, partial, n_empty):
    """Rank-ordered query lists (two ascending runs) and, in partial mode,
    rows that see no key (horizon -1): the tile span is the tile's max horizon.
    130 empty rows make whole tile pairs (2 x 32 tokens at G = 4) keyless."""
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(11)
    hkv, dh, n, H = 8, 128, 3000, 32
    a = np.sort(rng.choice(n, 250, replace=False))
    b = np.sort(rng.choice(n, 200, replace=False))
    hz = np.concatenate([a, b])
    if partial:
        hz[:n_empty] = -1
    q = T.as_tensor(rng.standard_normal((hz.size, H, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    k = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    v = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    hzt = T.as_tensor(hz, device=cuda)
    if partial:
        out, ml = E.recompute_attn_partial(q, k, v, hzt, H, hkv, dh)
        ml = ml.cpu().numpy()
        e = n_empty
        assert np.all(ml[:e, :, 1] == 0) and np.all(np.isneginf(ml[:e, :, 0]))
        assert np.all(out[:e].float().cpu().numpy() == 0)
        rows = slice(e, None)
        # (max, sum) in natural units of the scaled logits: l * e^m == sum_j e^(s_j)
        qd, kd = q.double().cpu().numpy()[e:], k.double().cpu().numpy()
        for i in (0, 100, 300):
            r = e + i
            for h in (0, 13):
                s_ = qd[i, h] @ kd[: hz[r] + 1, h // (H // hkv)].T / np.sqrt(dh)
                mt = s_.max()
                assert ml[r, h, 1] * np.exp(ml[r, h, 0] - mt) == pytest.approx(np.exp(s_ - mt).sum(), rel=2e-2)
    else:
        out = E.recompute_attn(q, k, v, hzt, H, hkv, dh)
        rows = slice(0, None)
    got = out.double().cpu().numpy()[rows]
    want, _ = O.prefix_attention(q.double().cpu().numpy()[rows], k.double().cpu().numpy(), v.double().cpu().numpy(),
                                 hz[rows])
    assert np.max(np.abs(got - want)) <= 1e-2 * np.max(np.abs(want))


@pytest.mark.parametrize("partial", [False, True])
def test_recompute_attention_large_grid_tcgen05(T, cuda, partial):
    """k = 2600 at 32 q / 8 kv heads (a grid near two waves, so the key-split
    path of the tcgen05 kernel is exercised): compare with the SIMT kernel on
    every row and with the oracle on sampled rows."""
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(5)
    hkv, dh, n, H, k = 8, 128, 6000, 32, 2600
    hz = np.sort(rng.choice(n, k, replace=False))
    if partial:
        hz[:70] = -1  # keyless rows (and one keyless tile pair) of the sharded partial mode
    q = T.as_tensor(rng.standard_normal((k, H, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    kk = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    vv = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    hzt = T.as_tensor(hz, device=cuda)
    if partial:
        tc, ml = E.recompute_attn_partial(q, kk, vv, hzt, H, hkv, dh)
        assert np.all(ml[:70].cpu().numpy()[..., 1] == 0)
    else:
        tc = E.recompute_attn(q, kk, vv, hzt, H, hkv, dh)
    simt = E.recompute_attn(q, kk, vv, hzt, H, hkv, dh, impl="simt") if not partial else None
    got = tc.double().cpu().numpy()
    rows = np.arange(70 if partial else 0, k)
    if simt is not None:
        ref = simt.double().cpu().numpy()
        assert np.max(np.abs(got - ref)) <= 1e-2 * np.max(np.abs(ref))
    pick = rows[rng.choice(rows.size, 40, replace=False)]
    want, _ = O.prefix_attention(q.double().cpu().numpy()[pick], kk.double().cpu().numpy(),
                                 vv.double().cpu().numpy(), hz[pick])
    assert np.max(np.abs(got[pick] - want)) <= 1e-2 * np.max(np.abs(want))
    if partial:
        assert np.all(got[:70] == 0)


@pytest.mark.parametrize("H,hkv,k", [(28, 4, 300), (28, 4, 2600), (24, 8, 2600)])
def test_recompute_attention_gqa_groups_not_dividing_128(T, cuda, H, hkv, k):
    """G = 7 (Qwen2.5-VL: 18 tokens x 7 heads = 126 rows per tile) and G = 3
    (42 tokens x 3 heads) on the tcgen05 kernel against the oracle on sampled
    rows."""
    from paper_2603_05353_b200 import engine as E

    rng = np.random.default_rng(H + k)
    dh, n = 128, 5000
    hz = np.sort(rng.choice(n, k, replace=False))
    q = T.as_tensor(rng.standard_normal((k, H, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    kk = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    vv = T.as_tensor(rng.standard_normal((n, hkv, dh)), dtype=T.float32).to(cuda, T.bfloat16)
    got = E.recompute_attn(q, kk, vv, T.as_tensor(hz, device=cuda), H, hkv, dh).double().cpu().numpy()
    pick = np.sort(rng.choice(k, 40, replace=False))
    want, _ = O.prefix_attention(q.double().cpu().numpy()[pick], kk.double().cpu().numpy(),
                                 vv.double().cpu().numpy(), hz[pick])
    assert np.max(np.abs(got[pick] - want)) <= 1e-2 * np.max(np.abs(want))


def test_stream_handle_follows_torch_current_stream(T, cuda):
    from paper_2603_05353_b200 import _native as N

    assert N.stream_handle() == T.cuda.current_stream().cuda_stream
    s = T.cuda.Stream()
    with T.cuda.stream(s):
        assert N.stream_handle() == s.cuda_stream
    assert N.stream_handle() == T.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("P,R,K,N", [(3, 32, 4096, 6144), (3, 32, 14336, 4096), (1, 32, 512, 1536),
                                     (3, 64, 512, 3584), (2, 96, 1024, 256)])
def test_prompt_mm_weight_stream_gemm(T, cuda, P, R, K, N):
    """ifkv_prompt_mm (tcgen05, K-major "out x in" weight operand, K splits)
    against an fp64 product of the same bf16 operands: fp32 accumulation only."""
    from paper_2603_05353_b200 import _native as NV
    from paper_2603_05353_b200 import engine as E

    g = T.Generator(device="cuda").manual_seed(P * 1000 + R)
    x = T.randn(P, R, K, device="cuda", generator=g).to(T.bfloat16)
    w = (T.randn(K, N, device="cuda", generator=g) / math.sqrt(K)).to(T.bfloat16)
    want = sum(x[p].double() @ w.double() for p in range(P))

    def rel(got):
        return float((got - want).abs().max() / want.abs().max())

    # tolerance: fp32 accumulation over K, calibrated on cuBLAS's own error
    # for the same bf16 operands (~1e-5 at K = 14336)
    cub = rel(sum(T.mm(x[p], w, out_dtype=T.float32).double() for p in range(P)))
    tol = max(1e-5, 2 * cub)
    wt = w.t().contiguous()  # the device layout: [N][K]
    for s in sorted({1, E.prompt_mm_splits(N, K, R, 148, P), min(K // 64, 7)}):
        out = T.full((s, R, N), float("nan"), dtype=T.float32, device="cuda")
        NV.call("ifkv_prompt_mm", NV.ptr(x), P, R, K, NV.ptr(wt), N, s, NV.ptr(out), NV.stream_handle())
        assert rel(out.double().sum(0)) < tol, (s, cub)
    assert rel(E.mm_parts(x, wt).double().sum(0)) < tol
    from paper_2603_05353_b200.errors import ConfigurationError

    with pytest.raises(ConfigurationError):
        NV.call("ifkv_prompt_mm", NV.ptr(x), P, 16, K, NV.ptr(w), N, 1, NV.ptr(out), NV.stream_handle())


def test_merge_partials_matches_state_merge(T, cuda):
    """ifkv_merge_partials (the chunk-sharded recompute's per-layer merge)
    against the torch softmax-state merge, including keyless partials."""
    from paper_2603_05353_b200 import engine as E
    from paper_2603_05353_b200 import sharding as SH

    g = T.Generator(device="cuda").manual_seed(3)
    P, S, H, Dh = 3, 37, 4, 128
    o = T.randn(P, S, H, Dh, device="cuda", generator=g).to(T.bfloat16)
    m = T.randn(P, S, H, device="cuda", generator=g) * 4
    l = T.rand(P, S, H, device="cuda", generator=g) * 10 + 0.1
    m[1, :5] = -float("inf")  # rank 1 saw no key for these queries
    l[1, :5] = 0.0
    ml = T.stack([m, l], dim=-1)
    got = E.merge_partials(o, ml).float()
    want = SH.merge_query_states(list(o), list(ml)).float()
    assert float((got - want).abs().max() / want.abs().max()) < 1e-2


def test_merge_prompt_states_matches_state_merge(T, cuda):
    """ifkv_merge_prompt_states (the chunk-sharded scoring pass's per-layer
    merge) against the torch merge, including ranks that saw no key."""
    from paper_2603_05353_b200 import engine as E
    from paper_2603_05353_b200 import sharding as SH

    g = T.Generator(device="cuda").manual_seed(4)
    P, G, M, H, Dh = 3, 2, 32, 8, 128
    ctx = T.randn(P, G, M, H, Dh, device="cuda", generator=g)
    m = T.randn(P, G, H, M, device="cuda", generator=g) * 3
    l = T.rand(P, G, H, M, device="cuda", generator=g) * 5 + 0.1
    m[2, :, :3] = -float("inf")
    l[2, :, :3] = 0.0
    ml = T.stack([m, l], dim=-1)
    got_c, got_ml = E.merge_prompt_states(ctx, ml)
    want_c, want_ml = SH.merge_prompt_states(list(ctx), list(ml))
    assert float((got_c - want_c).abs().max() / want_c.abs().max()) < 1e-5
    assert T.allclose(got_ml, want_ml, rtol=1e-5, atol=0)
