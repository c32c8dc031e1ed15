"""Recomputation-target selection (reference selection.py:1-322).

Attention-norm scoring runs the prompt forward on top of the assembled cache
with every context key read at the geometry's position.  The rotation is not
applied to the keys: the scorer folds R(delta) into the prompt queries of
each constant-delta run (q . R(d) k == (R(-d) q) . k), so it reads the stored
bf16 keys exactly and stays fp32-accurate.  The capture layer's post-softmax
mass is summed per context column on the device (``ifkv_score_columns``) and
the top-k is an exact radix select with the reference's tie rule
(``ifkv_topk_segments``).

Scores and selected indices stay on the device (``SelectionResult.scores``
fp32, ``.selected`` int64, ascending); ``scores_numpy()`` / ``selected_numpy()``
copy them to the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import Optional, Sequence, Union

import numpy as np

from . import engine as E
from .cache import AssembledCache
from .errors import ConfigurationError
from .positions import ChunkSpec, GeometryConfig, GeometryMode, PositionAssignment, assign_positions


def _torch():
    import torch

    return torch


class Strategy(Enum):
    ATTENTION_NORM = "attention-norm"
    CACHEBLEND = "cacheblend"
    EPIC = "epic"
    RANDOM = "random"

    @classmethod
    def parse(cls, name) -> "Strategy":
        if isinstance(name, cls):
            return name
        key = str(name).strip().lower().replace("_", "-")
        for s in cls:
            if s.value == key:
                return s
        raise ConfigurationError(f"unknown strategy {name!r}; expected one of " + ", ".join(s.value for s in cls))


def default_norm_layer(n_layers: int) -> int:
    """min(L - 1, floor(0.6 L)) (selection.py:48-50)."""
    return min(n_layers - 1, int(math.floor(0.6 * n_layers)))


@dataclass
class SelectionConfig:
    """Exactly one of topk / ratio; ratio resolves to ceil(ratio * N)
    (selection.py:53-87)."""

    strategy: Strategy = Strategy.ATTENTION_NORM
    topk: Optional[int] = None
    ratio: Optional[float] = None
    norm_layer: Optional[int] = None
    geometry: Union[GeometryConfig, GeometryMode, str, None] = None
    seed: int = 0
    cacheblend_layers: int = 2
    head_aggregation: str = "mean_over_heads"
    # attention-norm scores: "fp32" (fp32-accurate tcgen05 scorer, the fast
    # path) or "fp64" (exact.py: the scoring pass in float64, for selected
    # sets identical to the float64 reference at any boundary margin)
    score_precision: str = "fp32"

    def __post_init__(self):
        self.strategy = Strategy.parse(self.strategy)
        if (self.topk is None) == (self.ratio is None):
            raise ConfigurationError("exactly one of topk or ratio must be set")
        if self.ratio is not None and not 0.0 <= self.ratio <= 1.0:
            raise ConfigurationError(f"ratio must be in [0, 1], got {self.ratio}")
        if self.topk is not None and self.topk < 0:
            raise ConfigurationError(f"topk must be >= 0, got {self.topk}")
        if self.head_aggregation != "mean_over_heads":
            raise ConfigurationError(f"unsupported head aggregation {self.head_aggregation!r}")
        if self.score_precision not in ("fp32", "fp64"):
            raise ConfigurationError(f"score_precision must be 'fp32' or 'fp64', got {self.score_precision!r}")

    def resolve_budget(self, n_context: int) -> int:
        k = self.topk if self.topk is not None else math.ceil(self.ratio * n_context)
        if k > n_context:
            raise ConfigurationError(f"budget {k} exceeds context length {n_context}")
        return int(k)


@dataclass
class SelectionResult:
    scores: "object"  # fp32 [N] on device (or numpy for host-only strategies)
    selected: "object"  # int64 [k] ascending on device
    strategy: str
    geometry: Optional[str] = None
    budget: int = 0

    def __post_init__(self):
        self.budget = int(self.selected.shape[0])

    def scores_numpy(self) -> np.ndarray:
        s = self.scores
        return s.detach().double().cpu().numpy() if hasattr(s, "detach") else np.asarray(s, np.float64)

    def selected_numpy(self) -> np.ndarray:
        s = self.selected
        return s.detach().cpu().numpy().astype(np.int64) if hasattr(s, "detach") else np.asarray(s, np.int64)


def score_from_attention(attention, n_context: int) -> np.ndarray:
    """Head-mean then prompt-row sum of the context columns (selection.py:108-124).
    Host utility for explicit attention arrays (the injection seam)."""
    a = np.asarray(attention, dtype=np.float64)
    if a.ndim == 3:
        a = a.mean(axis=0)
    if a.ndim != 2:
        raise ConfigurationError(f"attention must be 2-D or 3-D, got shape {a.shape}")
    if n_context > a.shape[1]:
        raise ConfigurationError(f"n_context {n_context} exceeds key count {a.shape[1]}")
    return a[:, :n_context].sum(axis=0)


def score_attention_norm(weights, cache: AssembledCache, prompt_token_ids, positions: PositionAssignment,
                         norm_layer: int, precision: str = "fp32"):
    """Prompt-conditioned importance of every context token (selection.py:127-169).
    Returns fp32 [N] on the device (float64 with precision "fp64", exact.py)."""
    cfg = weights.config
    if not 0 <= norm_layer < cfg.n_layers:
        raise ConfigurationError(f"norm_layer {norm_layer} outside [0, {cfg.n_layers})")
    if cache.n_layers != cfg.n_layers:
        raise ConfigurationError("cache layer count does not match model")
    n = cache.context_length
    target = positions.context_concat()
    if target.size != n:
        raise ConfigurationError(f"position assignment covers {target.size} context tokens, cache has {n}")
    prompt = np.asarray(prompt_token_ids, dtype=np.int64)
    if prompt.ndim != 1 or prompt.size == 0:
        raise ConfigurationError("token_ids must be a nonempty 1-D sequence")
    if prompt.min() < 0 or prompt.max() >= cfg.vocab_size:
        raise ConfigurationError("token id outside vocabulary")
    group = E.PromptGroup(prompt, np.asarray(positions.prompt_positions, np.int64),
                          E.segments_from_deltas(target - cache.row_positions[:n]))
    if precision == "fp64":
        from .exact import prompt_scores_f64

        return prompt_scores_f64(weights, cache.keys, cache.values, [group], norm_layer)[:n]
    out = E.prompt_forward(weights, cache.keys, cache.values, [group], capture_layer=norm_layer)
    return out.scores[:n]


def select_topk(scores, k: int):
    """Indices of the k largest scores, ties to the lower index, ascending
    (selection.py:172-183).  Device int64 tensor, tagged as a valid recompute
    plan (sorted, unique, in range) for ``make_plan``.

    fp32 scores (attention-norm) run the exact radix select
    (``ifkv_topk_segments``); fp64 scores (the CacheBlend baseline, summed in
    fp64) keep their precision: a stable descending sort on the device, so
    near-equal fp64 scores are not collapsed into fp32 ties."""
    torch = _torch()
    if not isinstance(scores, torch.Tensor):
        a = np.asarray(scores)
        scores = torch.as_tensor(a, dtype=torch.float64 if a.dtype == np.float64 else torch.float32, device="cuda")
    n = scores.numel()
    if k > n:
        raise ConfigurationError(f"k ({k}) exceeds score count ({n})")
    if k < 0:
        raise ConfigurationError(f"k must be >= 0, got {k}")
    if k == 0:
        idx = torch.zeros(0, dtype=torch.int64, device=scores.device)
    elif scores.dtype == torch.float64:
        order = torch.sort(scores.contiguous(), descending=True, stable=True).indices[:k]
        idx = torch.sort(order).values
    else:
        idx, _, _ = E.topk_segments(scores.to(torch.float32).contiguous(), [0, n], [k])
    idx._ifkv_valid_plan = n  # produced here: sorted, unique, in [0, n)
    return idx


def score_cacheblend(weights, chunks: Sequence[ChunkSpec], early_layers: int):
    """CacheBlend baseline (selection.py:190-223): per context token, the L2
    distance between its block outputs in the chunk-local runs (positions
    0..len-1, causal inside the chunk) and in one full-context causal run,
    summed over the first ``early_layers`` layers.  Both runs go through the
    layer stack (chunk-local runs one chunk at a time into a scratch slab);
    the distances accumulate on the device in fp64 (``ifkv_row_dist_accum``).
    Returns fp64 [N] on the device."""
    torch = _torch()
    cfg = weights.config
    if early_layers < 1:
        raise ConfigurationError("early_layers must be >= 1")
    if early_layers > cfg.n_layers:
        raise ConfigurationError(f"early_layers {early_layers} exceeds n_layers {cfg.n_layers}")
    if not chunks:
        raise ConfigurationError("no chunks to score")
    dev = weights.device
    lens = [int(np.asarray(c.token_ids).size) for c in chunks]
    n = sum(lens)
    if n > cfg.max_position:
        raise ConfigurationError(f"context length {n} exceeds max_position {cfg.max_position}")
    toks = np.concatenate([np.asarray(c.token_ids, np.int64) for c in chunks])
    if toks.min() < 0 or toks.max() >= cfg.vocab_size:
        raise ConfigurationError("token id outside vocabulary")
    local = torch.empty((early_layers, n, cfg.d_model), dtype=torch.float32, device=dev)
    kv_shape = (early_layers, max(lens), cfg.kv_heads, cfg.d_head)
    ks = torch.empty(kv_shape, dtype=weights.torch_dtype, device=dev)
    vs = torch.empty_like(ks)
    r0 = 0
    for c, ln in zip(chunks, lens):
        ar = torch.arange(ln, dtype=torch.int64, device=dev)
        ids = E.h2d(np.asarray(c.token_ids, np.int64), dev)
        E.layer_stack(weights, ids, ar, ks, vs, ar, ar, n_layers=early_layers,
                      on_hidden=lambda li, h, r0=r0, ln=ln: local[li, r0:r0 + ln].copy_(h))
        r0 += ln
    del ks, vs
    kf = torch.empty((early_layers, n, cfg.kv_heads, cfg.d_head), dtype=weights.torch_dtype, device=dev)
    vf = torch.empty_like(kf)
    ar = torch.arange(n, dtype=torch.int64, device=dev)
    scores = torch.zeros(n, dtype=torch.float64, device=dev)
    E.layer_stack(weights, E.h2d(toks, dev), ar, kf, vf, ar, ar, n_layers=early_layers,
                  on_hidden=lambda li, h: E.row_dist_accum(local[li], h, scores))
    return scores


def select_epic(chunk_lengths: Sequence[int], ratio: float) -> np.ndarray:
    """First ceil(ratio * len) tokens of every chunk (selection.py:226-239)."""
    if not 0.0 <= ratio <= 1.0:
        raise ConfigurationError(f"ratio must be in [0, 1], got {ratio}")
    starts = np.concatenate([[0], np.cumsum(chunk_lengths)[:-1]]) if len(chunk_lengths) else []
    out = [s + np.arange(math.ceil(ratio * n), dtype=np.int64) for s, n in zip(starts, chunk_lengths)]
    return np.concatenate(out).astype(np.int64) if out else np.zeros(0, np.int64)


def select_random(n: int, k: int, seed: int) -> np.ndarray:
    """Uniform k-of-n without replacement, deterministic per seed (selection.py:242-255)."""
    if k > n:
        raise ConfigurationError(f"k ({k}) exceeds context length ({n})")
    if k < 0:
        raise ConfigurationError(f"k must be >= 0, got {k}")
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=k, replace=False).astype(np.int64))


def resolve_geometry(config: SelectionConfig, cache: AssembledCache, prompt_length: int, max_position: int):
    geometry = config.geometry if config.geometry is not None else GeometryMode.GLOBAL
    if not isinstance(geometry, GeometryConfig):
        geometry = GeometryConfig(mode=GeometryMode.parse(geometry), prompt_length=prompt_length,
                                  chunk_lengths=tuple(cache.chunk_lengths), max_position=max_position)
    return geometry


def run_selection(weights, chunks: Sequence[ChunkSpec], cache: AssembledCache, prompt_token_ids,
                  config: SelectionConfig) -> SelectionResult:
    """Strategy dispatch (selection.py:263-322)."""
    torch = _torch()
    n = cache.context_length
    prompt = np.asarray(prompt_token_ids, dtype=np.int64)
    if config.strategy is Strategy.ATTENTION_NORM:
        geometry = resolve_geometry(config, cache, int(prompt.size), weights.config.max_position)
        assignment = assign_positions(geometry, chunks)
        nl = config.norm_layer if config.norm_layer is not None else default_norm_layer(weights.config.n_layers)
        scores = score_attention_norm(weights, cache, prompt, assignment, nl, config.score_precision)
        k = config.resolve_budget(n)
        return SelectionResult(scores=scores, selected=select_topk(scores, k), strategy=config.strategy.value,
                               geometry=geometry.mode.value)
    dev = cache.keys.device
    if config.strategy is Strategy.EPIC:
        ratio = config.ratio if config.ratio is not None else config.topk / max(n, 1)
        sel = select_epic(cache.chunk_lengths, ratio)
    elif config.strategy is Strategy.RANDOM:
        sel = select_random(n, config.resolve_budget(n), config.seed)
    else:  # CacheBlend
        if not chunks:
            raise ConfigurationError("no chunks to score")
        scores = score_cacheblend(weights, chunks, config.cacheblend_layers)
        return SelectionResult(scores=scores, selected=select_topk(scores, config.resolve_budget(n)),
                               strategy=config.strategy.value)
    scores = np.zeros(n, np.float32)
    scores[sel] = 1.0
    return SelectionResult(scores=torch.as_tensor(scores, device=dev), selected=torch.as_tensor(sel, device=dev),
                           strategy=config.strategy.value)
