"""Model configuration and weights (host and HBM-resident).

Mirrors the reference's ``ModelConfig`` / ``Weights`` / ``init_weights``
(model.py:41-218) and adds grouped-query attention (``n_kv_heads``): the
reference is MHA-only, the benchmark shapes (Llama-3-8B, Qwen2.5-VL-7B) are
GQA.  With ``n_kv_heads`` unset the draw order and shapes are exactly the
reference's, so ``init_weights`` reproduces its tensors bit for bit.

``DeviceWeights`` is the HBM layout the kernels read: every projection is
stored "out x in" (W^T of the reference's x @ W, row-major [N][K]) so both
GEMM operands are K-major for the tcgen05 kernels: per layer one fused
[(H + 2 Hkv) Dh, d] QKV matrix, the O projection [d, d], one fused
[2 d_ff, d] gate|up matrix whose rows interleave gate and up in blocks of
``gu_block`` (64: gate j..j+63, up j..j+63, ... -- the SwiGLU epilogue pairs
g_j with u_j inside one tile) and the down projection [d, d_ff]; bf16 (perf)
or fp32 (parity mode); norm gains stay fp32.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .errors import ConfigurationError

PRECISIONS = ("bf16", "f32")
HOST_PRECISIONS = {"f32": np.float32, "f64": np.float64}


@dataclass(frozen=True)
class ModelConfig:
    """Decoder dimensions; d_model == n_heads * d_head (model.py:41-72)."""

    n_layers: int
    n_heads: int
    d_model: int
    d_head: int
    d_ff: int
    vocab_size: int
    rope_base: float = 10000.0
    max_position: int = 8192
    n_kv_heads: Optional[int] = None

    def __post_init__(self):
        checks = [
            (self.n_layers >= 1, f"n_layers must be >= 1, got {self.n_layers}"),
            (self.n_heads >= 1, f"n_heads must be >= 1, got {self.n_heads}"),
            (self.vocab_size >= 2, f"vocab_size must be >= 2, got {self.vocab_size}"),
            (self.d_head >= 2 and self.d_head % 2 == 0, f"d_head must be a positive even number, got {self.d_head}"),
            (self.d_model == self.n_heads * self.d_head,
             f"d_model ({self.d_model}) must equal n_heads*d_head ({self.n_heads * self.d_head})"),
            (self.d_ff >= 1, f"d_ff must be >= 1, got {self.d_ff}"),
            (self.max_position >= 1, f"max_position must be >= 1, got {self.max_position}"),
            (self.rope_base > 0, f"rope_base must be positive, got {self.rope_base}"),
        ]
        if self.n_kv_heads is not None:
            checks.append((self.n_kv_heads >= 1 and self.n_heads % self.n_kv_heads == 0,
                           f"n_kv_heads ({self.n_kv_heads}) must divide n_heads ({self.n_heads})"))
        for ok, msg in checks:
            if not ok:
                raise ConfigurationError(msg)

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.d_head

    def params_per_layer(self) -> int:
        d = self.d_model
        return d * d * 2 + 2 * d * self.kv_dim + 3 * d * self.d_ff


# ---------------------------------------------------------------------------
# Named shapes (BASELINE.json configs)
# ---------------------------------------------------------------------------


def c1_config() -> ModelConfig:
    """BASELINE config 1: tiny random-init Llama, Dh = 128."""
    return ModelConfig(n_layers=2, n_heads=4, d_model=512, d_head=128, d_ff=1792, vocab_size=1024,
                       rope_base=10000.0, max_position=8192)


def llama3_8b_config(max_position: int = 262144) -> ModelConfig:
    """Llama-3-8B shape: 32 layers, 32 q / 8 kv heads, d_ff 14336, RoPE 5e5."""
    return ModelConfig(n_layers=32, n_heads=32, d_model=4096, d_head=128, d_ff=14336, vocab_size=128256,
                       rope_base=500000.0, max_position=max_position, n_kv_heads=8)


def qwen25vl_7b_config(max_position: int = 262144) -> ModelConfig:
    """Qwen2.5-VL-7B language-model shape (1-D RoPE)."""
    return ModelConfig(n_layers=28, n_heads=28, d_model=3584, d_head=128, d_ff=18944, vocab_size=152064,
                       rope_base=1000000.0, max_position=max_position, n_kv_heads=4)


def toy_config(n_layers=4, n_heads=4, d_head=16, d_ff=256, vocab_size=256, max_position=16384,
               rope_base=10000.0) -> ModelConfig:
    """Desk-scale dimensions (harness.py:102-121)."""
    return ModelConfig(n_layers=n_layers, n_heads=n_heads, d_model=n_heads * d_head, d_head=d_head, d_ff=d_ff,
                       vocab_size=vocab_size, rope_base=rope_base, max_position=max_position)


# ---------------------------------------------------------------------------
# Host weights (model.py:75-218)
# ---------------------------------------------------------------------------


@dataclass
class LayerWeights:
    attn_norm: np.ndarray
    wq: np.ndarray  # (d, H*Dh)
    wk: np.ndarray  # (d, Hkv*Dh)
    wv: np.ndarray
    wo: np.ndarray  # (d, d)
    mlp_norm: np.ndarray
    w_gate: np.ndarray  # (d, d_ff)
    w_up: np.ndarray
    w_down: np.ndarray  # (d_ff, d)

    FIELDS = ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "w_gate", "w_up", "w_down")

    def tensors(self):
        return [(n, getattr(self, n)) for n in self.FIELDS]


@dataclass
class Weights:
    """Host (NumPy) weights; the oracle and the reference read these."""

    config: ModelConfig
    embedding: np.ndarray
    layers: List[LayerWeights]
    final_norm: np.ndarray
    out_head: np.ndarray
    _fingerprint: Optional[int] = field(default=None, repr=False, compare=False)

    @property
    def dtype(self):
        return self.embedding.dtype

    def named_tensors(self):
        yield "embedding", self.embedding
        for i, lw in enumerate(self.layers):
            for n, t in lw.tensors():
                yield f"layer{i}.{n}", t
        yield "final_norm", self.final_norm
        yield "out_head", self.out_head

    def fingerprint(self) -> int:
        """64-bit blake2b identity of config, precision and tensor bytes."""
        if self._fingerprint is None:
            c = self.config
            h = hashlib.blake2b(digest_size=8)
            h.update(struct.pack("<8qd", c.n_layers, c.n_heads, c.kv_heads, c.d_model, c.d_head, c.d_ff,
                                 c.vocab_size, c.max_position, c.rope_base))
            h.update(str(self.dtype).encode())
            for name, t in self.named_tensors():
                h.update(name.encode())
                h.update(np.ascontiguousarray(t).tobytes())
            self._fingerprint = int.from_bytes(h.digest(), "little")
        return self._fingerprint

    def astype(self, dtype) -> "Weights":
        cast = lambda a: np.asarray(a).astype(dtype)  # noqa: E731
        return Weights(self.config, cast(self.embedding),
                       [LayerWeights(**{n: cast(t) for n, t in lw.tensors()}) for lw in self.layers],
                       cast(self.final_norm), cast(self.out_head))

    def bf16_rounded(self) -> "Weights":
        """Round every tensor to the nearest bf16 value (kept in float64)."""
        return Weights(self.config, bf16_round(self.embedding),
                       [LayerWeights(**{n: bf16_round(t) for n, t in lw.tensors()}) for lw in self.layers],
                       bf16_round(self.final_norm), bf16_round(self.out_head))


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def init_weights(config: ModelConfig, seed: int, precision: str = "f64") -> Weights:
    """Deterministic Gaussian init in the reference's draw order (model.py:171-218).

    PCG64(seed) draws, in float64: embedding (V, d); per layer wq, wk, wv, wo,
    w_gate, w_up, w_down; then out_head.  Projections scale by 1/sqrt(fan_in)
    (d, or d_ff for w_down); norm gains are ones.  For GQA configs wk/wv are
    (d, Hkv*Dh).
    """
    if precision not in HOST_PRECISIONS:
        raise ConfigurationError(f"unknown precision {precision!r}, expected one of {sorted(HOST_PRECISIONS)}")
    rng = np.random.default_rng(seed)
    d, dff, v, kv = config.d_model, config.d_ff, config.vocab_size, config.kv_dim
    s_in = 1.0 / np.sqrt(d)
    s_down = 1.0 / np.sqrt(dff)
    embedding = rng.standard_normal((v, d))
    layers = []
    for _ in range(config.n_layers):
        wq = rng.standard_normal((d, d)) * s_in
        wk = rng.standard_normal((d, kv)) * s_in
        wv = rng.standard_normal((d, kv)) * s_in
        wo = rng.standard_normal((d, d)) * s_in
        wg = rng.standard_normal((d, dff)) * s_in
        wu = rng.standard_normal((d, dff)) * s_in
        wd = rng.standard_normal((dff, d)) * s_down
        layers.append(LayerWeights(np.ones(d), wq, wk, wv, wo, np.ones(d), wg, wu, wd))
    out_head = rng.standard_normal((d, v)) * s_in
    w = Weights(config, embedding, layers, np.ones(d), out_head)
    return w if precision == "f64" else w.astype(HOST_PRECISIONS[precision])


# ---------------------------------------------------------------------------
# HBM-resident weights
# ---------------------------------------------------------------------------


def gu_block_for(d_ff: int) -> int:
    """Gate/up interleave block of the fused gate|up weight: 64 when it
    divides d_ff (the SwiGLU GEMM epilogue's unit), else d_ff ([gate; up])."""
    return 64 if d_ff % 64 == 0 else d_ff


def interleave_gu(gate_t, up_t, block: int):
    """[d_ff, d] gate^T and up^T -> [2 d_ff, d] rows (gate block, up block)*.
    Works for numpy arrays and torch tensors."""
    dff, d = gate_t.shape
    nb = dff // block
    if hasattr(gate_t, "new_empty"):  # torch
        import torch

        return torch.stack([gate_t.reshape(nb, block, d), up_t.reshape(nb, block, d)], 1).reshape(2 * dff, d)
    return np.stack([gate_t.reshape(nb, block, d), up_t.reshape(nb, block, d)], 1).reshape(2 * dff, d)


def deinterleave_gu(gu_t, block: int):
    """Inverse of interleave_gu: -> (gate^T, up^T)."""
    two_dff, d = gu_t.shape
    dff = two_dff // 2
    v = gu_t.reshape(dff // block, 2, block, d)
    return v[:, 0].reshape(dff, d), v[:, 1].reshape(dff, d)


@dataclass
class DeviceLayer:
    attn_norm: "object"  # torch fp32 [d]
    wqkv: "object"  # [(H + 2 Hkv) Dh, d] = [wq | wk | wv]^T
    wo: "object"  # [d, d] = wo^T
    mlp_norm: "object"
    wgu: "object"  # [2 d_ff, d]: gate^T / up^T rows interleaved in gu_block blocks
    wdown: "object"  # [d, d_ff] = w_down^T


@dataclass
class DeviceWeights:
    config: ModelConfig
    precision: str  # "bf16" | "f32"
    embedding: "object"
    layers: List[DeviceLayer]
    final_norm: "object"
    out_head: "object"  # [vocab, d] = out_head^T
    fingerprint_value: int = 0

    @property
    def gu_block(self) -> int:
        return gu_block_for(self.config.d_ff)

    def fingerprint(self) -> int:
        return self.fingerprint_value

    @property
    def torch_dtype(self):
        import torch

        return torch.bfloat16 if self.precision == "bf16" else torch.float32

    @property
    def device(self):
        return self.embedding.device

    @classmethod
    def from_host(cls, weights: Weights, precision: str = "bf16", device="cuda") -> "DeviceWeights":
        """Upload host weights (rounded to bf16 in bf16 mode)."""
        import torch

        if precision not in PRECISIONS:
            raise ConfigurationError(f"unknown device precision {precision!r}, expected one of {PRECISIONS}")
        dt = torch.bfloat16 if precision == "bf16" else torch.float32

        def up(a, dtype=dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device=device, dtype=dtype)

        blk = gu_block_for(weights.config.d_ff)
        layers = []
        for lw in weights.layers:
            layers.append(DeviceLayer(
                attn_norm=up(lw.attn_norm, torch.float32),
                wqkv=up(np.concatenate([lw.wq, lw.wk, lw.wv], axis=1).T),
                wo=up(np.asarray(lw.wo).T),
                mlp_norm=up(lw.mlp_norm, torch.float32),
                wgu=up(interleave_gu(np.asarray(lw.w_gate).T, np.asarray(lw.w_up).T, blk)),
                wdown=up(np.asarray(lw.w_down).T),
            ))
        return cls(weights.config, precision, up(weights.embedding), layers, up(weights.final_norm, torch.float32),
                   up(np.asarray(weights.out_head).T), fingerprint_value=weights.fingerprint())

    @classmethod
    def random(cls, config: ModelConfig, seed: int, precision: str = "bf16", device="cuda") -> "DeviceWeights":
        """Same-distribution init drawn on the GPU (perf shapes: drawing 8 B
        float64 values on the host as init_weights does is infeasible)."""
        import torch

        dt = torch.bfloat16 if precision == "bf16" else torch.float32
        gen = torch.Generator(device=device)
        gen.manual_seed(seed)
        d, dff, kv = config.d_model, config.d_ff, config.kv_dim

        def draw(shape, scale):
            out = torch.empty(shape, dtype=dt, device=device)
            rows = max(1, (1 << 26) // shape[1])
            for r0 in range(0, shape[0], rows):
                blk = torch.randn((min(rows, shape[0] - r0), shape[1]), generator=gen, device=device,
                                  dtype=torch.float32)
                out[r0:r0 + blk.shape[0]] = (blk * scale).to(dt)
            return out

        s_in, s_down = 1.0 / np.sqrt(d), 1.0 / np.sqrt(dff)
        emb = draw((config.vocab_size, d), 1.0)
        layers = []
        for _ in range(config.n_layers):  # i.i.d. draws: stored directly in the "out x in" layout
            layers.append(DeviceLayer(
                attn_norm=torch.ones(d, dtype=torch.float32, device=device),
                wqkv=draw((d + 2 * kv, d), s_in),
                wo=draw((d, d), s_in),
                mlp_norm=torch.ones(d, dtype=torch.float32, device=device),
                wgu=draw((2 * dff, d), s_in),
                wdown=draw((d, dff), s_down),
            ))
        head = draw((config.vocab_size, d), s_in)
        h = hashlib.blake2b(repr((config, seed, precision, "device-random")).encode(), digest_size=8)
        return cls(config, precision, emb, layers, torch.ones(d, dtype=torch.float32, device=device), head,
                   fingerprint_value=int.from_bytes(h.digest(), "little"))

    def to_host(self) -> Weights:
        """Exact float64 copy of the device values (the oracle's weights)."""
        import torch

        c = self.config
        hd = lambda t: t.detach().to(torch.float64).cpu().numpy()  # noqa: E731
        ht = lambda t: np.ascontiguousarray(hd(t).T)  # noqa: E731  ("out x in" -> the reference's [in, out])
        qd, kvd = c.d_model, c.kv_dim
        layers = []
        for dl in self.layers:
            qkv = ht(dl.wqkv)
            g_t, u_t = deinterleave_gu(hd(dl.wgu), self.gu_block)
            layers.append(LayerWeights(hd(dl.attn_norm), qkv[:, :qd], qkv[:, qd:qd + kvd], qkv[:, qd + kvd:],
                                       ht(dl.wo), hd(dl.mlp_norm), np.ascontiguousarray(g_t.T),
                                       np.ascontiguousarray(u_t.T), ht(dl.wdown)))
        return Weights(c, hd(self.embedding), layers, hd(self.final_norm), ht(self.out_head))
