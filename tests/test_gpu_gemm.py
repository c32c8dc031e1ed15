"""The tcgen05 CTA-pair projection GEMM (csrc/tc_gemm.cu) and its fused
epilogues against a plain PyTorch fp32 reference of the same bf16 operands.

Reference arithmetic: x @ wq/wk/wv + RoPE + K/V scatter (recompute.py:98-112,
cache.py:354-363), h += ctx @ wo and h += a @ w_down (model.py:448-452),
silu(x @ w_gate) * (x @ w_up) (model.py:283-294)."""

import math

import pytest

pytestmark = pytest.mark.gpu

TILES = (0, 1256, 1224, 1192, 1160, 1128)


def _rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("M,K,N", [(1, 64, 128), (5, 16, 96), (300, 512, 768), (257, 1024, 640), (700, 96, 200),
                                   (1000, 4096, 1536)])
def test_gemm_plain_f32_and_residual(T, cuda, M, K, N):
    from paper_2603_05353_b200 import _native as NV

    g = T.Generator(device="cuda").manual_seed(M * 7 + K)
    a = T.randn(M, K, device="cuda", generator=g).to(T.bfloat16)
    w = (T.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(T.bfloat16)
    ref = a.float() @ w.float().t()
    for tile in TILES:
        o16 = T.empty(M, N, dtype=T.bfloat16, device="cuda")
        o32 = T.full((M, N), float("nan"), device="cuda")
        h = T.randn(M, N, device="cuda", generator=g)
        h0 = h.clone()
        s = NV.stream_handle()
        NV.call("ifkv_gemm", NV.ptr(a), K, M, K, NV.ptr(w), N, NV.IFKV_BF16, NV.ptr(o16), N, 0, tile, s)
        NV.call("ifkv_gemm", NV.ptr(a), K, M, K, NV.ptr(w), N, NV.IFKV_F32, NV.ptr(o32), N, 0, tile, s)
        NV.call("ifkv_gemm", NV.ptr(a), K, M, K, NV.ptr(w), N, NV.IFKV_F32, NV.ptr(h), N, 1, tile, s)
        assert _rel(o16, ref) < 8e-3, tile  # bf16 output rounding
        assert _rel(o32, ref) < 2e-5, tile  # fp32 accumulation only
        assert _rel(h - h0, ref) < 2e-5, tile


def test_gemm_strided_operand_and_output(T, cuda):
    """lda > K (a column slice of a wider activation) and ldo > N."""
    from paper_2603_05353_b200 import _native as NV

    g = T.Generator(device="cuda").manual_seed(5)
    big = T.randn(333, 640, device="cuda", generator=g).to(T.bfloat16)
    a = big[:, :512]
    w = (T.randn(384, 512, device="cuda", generator=g) / 22).to(T.bfloat16)
    out = T.zeros(333, 400, device="cuda")
    NV.call("ifkv_gemm", NV.ptr(a), 640, 333, 512, NV.ptr(w), 384, NV.IFKV_F32, NV.ptr(out), 400, 0, 0,
            NV.stream_handle())
    assert _rel(out[:, :384], a.float() @ w.float().t()) < 2e-5
    assert T.all(out[:, 384:] == 0)


@pytest.mark.parametrize("M", [37, 300, 1000])
def test_gemm_qkv_rope_scatter_epilogue(T, cuda, M):
    from paper_2603_05353_b200 import _native as NV

    H, Hkv, Dh, K, rows = 8, 2, 128, 512, 2048
    g = T.Generator(device="cuda").manual_seed(M)
    a = T.randn(M, K, device="cuda", generator=g).to(T.bfloat16)
    w = (T.randn((H + 2 * Hkv) * Dh, K, device="cuda", generator=g) / math.sqrt(K)).to(T.bfloat16)
    pos = T.randint(0, 100000, (M,), device="cuda", generator=g)
    cs = T.empty((M, Dh // 2, 2), dtype=T.float32, device="cuda")
    s = NV.stream_handle()
    NV.call("ifkv_rope_table", NV.ptr(pos), M, Dh, 500000.0, NV.ptr(cs), s)
    dst = T.randperm(rows, device="cuda", generator=g)[:M].contiguous()
    ref = (a.float() @ w.float().t()).view(M, H + 2 * Hkv, Dh // 2, 2)
    c, sn = cs[:, None, :, 0], cs[:, None, :, 1]
    x, y = ref[..., 0], ref[..., 1]
    rot = T.stack([x * c - y * sn, x * sn + y * c], -1).view(M, H + 2 * Hkv, Dh)
    for tile in (0, 1256, 1128):
        kd = T.zeros(rows, Hkv, Dh, dtype=T.bfloat16, device="cuda")
        vd = T.zeros_like(kd)
        q = T.empty(M, H, Dh, dtype=T.bfloat16, device="cuda")
        NV.call("ifkv_gemm_qkv_rope_scatter", NV.ptr(a), K, M, K, NV.ptr(w), H, Hkv, 0, NV.ptr(cs), NV.ptr(q),
                NV.ptr(kd), NV.ptr(vd), NV.ptr(dst), tile, s)
        assert _rel(q, rot[:, :H]) < 8e-3
        assert _rel(kd[dst], rot[:, H:H + Hkv]) < 8e-3
        assert _rel(vd[dst], ref.view(M, -1, Dh)[:, H + Hkv:]) < 8e-3
        untouched = T.ones(rows, dtype=T.bool, device="cuda")
        untouched[dst] = False
        assert T.all(kd[untouched] == 0) and T.all(vd[untouched] == 0)  # scatter writes only its rows
        # K/V-only projection (the last layer) writes the same rows bit for bit
        kd2, vd2 = T.zeros_like(kd), T.zeros_like(kd)
        NV.call("ifkv_gemm_qkv_rope_scatter", NV.ptr(a), K, M, K, NV.ptr(w[H * Dh:].contiguous()), H, Hkv, 1,
                NV.ptr(cs), None, NV.ptr(kd2), NV.ptr(vd2), NV.ptr(dst), tile, s)
        assert T.equal(kd2, kd) and T.equal(vd2, vd)


@pytest.mark.parametrize("M,K,dff", [(300, 512, 1792), (4916, 1024, 512), (33, 64, 64)])
def test_gemm_swiglu_epilogue(T, cuda, M, K, dff):
    from paper_2603_05353_b200 import _native as NV
    from paper_2603_05353_b200.model import interleave_gu

    g = T.Generator(device="cuda").manual_seed(dff)
    a = T.randn(M, K, device="cuda", generator=g).to(T.bfloat16)
    wg = (T.randn(dff, K, device="cuda", generator=g) / math.sqrt(K)).to(T.bfloat16)
    wu = (T.randn(dff, K, device="cuda", generator=g) / math.sqrt(K)).to(T.bfloat16)
    w = interleave_gu(wg, wu, 64).contiguous()
    ref = T.nn.functional.silu(a.float() @ wg.float().t()) * (a.float() @ wu.float().t())
    for tile in (0, 1256, 1128):
        out = T.zeros(M, dff, dtype=T.bfloat16, device="cuda")
        NV.call("ifkv_gemm_swiglu", NV.ptr(a), K, M, K, NV.ptr(w), dff, NV.ptr(out), tile, NV.stream_handle())
        assert _rel(out, ref) < 1e-2, tile
    # the unfused path (GEMM + ifkv_silu_mul on the interleaved layout) agrees
    from paper_2603_05353_b200 import engine as E

    gu = E.gemm(a, w)
    a2 = E.silu_mul(gu.unsqueeze(0), 1, dff, NV.OUT_BF16, 64)
    assert _rel(a2, ref) < 1e-2


def test_gemm_argument_errors(T, cuda):
    from paper_2603_05353_b200 import _native as NV
    from paper_2603_05353_b200.errors import ConfigurationError

    a = T.zeros(64, 100, dtype=T.bfloat16, device="cuda")
    w = T.zeros(128, 100, dtype=T.bfloat16, device="cuda")
    out = T.zeros(64, 128, dtype=T.bfloat16, device="cuda")
    with pytest.raises(ConfigurationError, match="multiples of 8"):  # K = 100: rows not 16-byte multiples
        NV.call("ifkv_gemm", NV.ptr(a), 100, 64, 100, NV.ptr(w), 128, NV.IFKV_BF16, NV.ptr(out), 128, 0, 0,
                NV.stream_handle())
    with pytest.raises(ConfigurationError, match="fp32"):  # accumulate into bf16
        NV.call("ifkv_gemm", NV.ptr(a), 96, 64, 96, NV.ptr(w), 128, NV.IFKV_BF16, NV.ptr(out), 128, 1, 0,
                NV.stream_handle())
    with pytest.raises(ConfigurationError, match="tile"):
        NV.call("ifkv_gemm", NV.ptr(a), 96, 64, 96, NV.ptr(w), 128, NV.IFKV_BF16, NV.ptr(out), 128, 0, 1300,
                NV.stream_handle())
    with pytest.raises(ConfigurationError, match="multiple of 64"):
        NV.call("ifkv_gemm_swiglu", NV.ptr(a), 96, 64, 96, NV.ptr(w), 48, NV.ptr(out), 0, NV.stream_handle())
