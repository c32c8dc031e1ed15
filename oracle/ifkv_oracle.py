"""NumPy restatement of InfoFlow-KV's query-time context-assembly path.

TEST INFRASTRUCTURE ONLY -- this module is the parity checker and the timed
CPU baseline ("port") for the B200 implementation in
``paper_2603_05353_b200``.  It must never be imported by the product package.

It restates, function by function, the algorithm of the reference package
``chunkkv`` 0.1.0 (pure Python/NumPy, mounted at /root/reference/pkg/src/chunkkv;
every function below cites the reference file:line it follows).  It differs from
the reference only where the reference's structure is unusable at benchmark
shapes, never in the arithmetic:

* grouped-query attention (``n_kv_heads`` < ``n_heads``) is native; with
  ``n_kv_heads == n_heads`` it is exactly the reference's MHA;
* attention is evaluated in blocks of query rows, so an (H, k, N) probability
  tensor is never materialised at once (the reference's dense masks need
  41 GB at 32K context);
* layers whose outputs cannot influence the requested result (the layers
  above the capture layer in scoring, the last layer's attention/MLP in
  recomputation) are skipped; their results are unused by the reference too.

Pinning: ``tests/golden/make_golden.py`` runs the reference itself in this
container and commits its outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this module against every fixture
(selected index sets and permutations bit-exact, floats to 1e-9).

Arithmetic runs in the dtype of the weights (float64 for parity, float32 for
the CPU baseline timing), exactly like the reference (model.py:13-17).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

RMS_EPS = 1e-6  # model.py:33
PREFILLED_LOCAL, RECOMPUTED_GLOBAL, FULL_PREFILL = 0, 1, 2  # cache.py:31-34
GEOMETRY_MODES = ("GLOBAL", "HL-HP", "HL-TP", "TL-TP")  # positions.py:32-36
CHUNK_SCORE_MODES = ("sum", "mean", "max")  # reorder.py:33

# Query-row block size for attention; keeps (H, rows, S) temporaries bounded.
_ATTN_BYTES_BUDGET = 1 << 29


class OracleError(ValueError):
    """Raised where the reference raises ConfigurationError (errors.py:5)."""


# ---------------------------------------------------------------------------
# model geometry helpers
# ---------------------------------------------------------------------------


def _kv_heads(cfg) -> int:
    return int(getattr(cfg, "n_kv_heads", None) or cfg.n_heads)


def _dtype(weights) -> np.dtype:
    return weights.embedding.dtype


# ---------------------------------------------------------------------------
# Rotary embedding (model.py:226-270)
# ---------------------------------------------------------------------------


def rope_theta(d_head: int, base: float) -> np.ndarray:
    """theta_i = base ** (-2 i / d) in float64 (model.py:226-231)."""
    if d_head < 2 or d_head % 2:
        raise OracleError(f"RoPE dimension must be even and >= 2, got {d_head}")
    return float(base) ** (-2.0 * np.arange(d_head // 2, dtype=np.float64) / d_head)


def rope_rotate(x: np.ndarray, positions, base: float) -> np.ndarray:
    """Rotate interleaved pairs (x[2i], x[2i+1]) of every head by theta_i * p_t.

    x is (T, heads, Dh); positions (T,) may be any real numbers (deltas are
    used to move stored keys).  Angles and trig in float64, result cast back
    to x's dtype (model.py:254-270).
    """
    x = np.asarray(x)
    t, _, dh = x.shape
    ang = np.asarray(positions, dtype=np.float64).reshape(t, 1, 1) * rope_theta(dh, base)[None, None, :]
    c, s = np.cos(ang), np.sin(ang)
    even, odd = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = even * c - odd * s
    out[..., 1::2] = even * s + odd * c
    return out


# ---------------------------------------------------------------------------
# Block primitives (model.py:278-315)
# ---------------------------------------------------------------------------


def rms_norm(x: np.ndarray, gain: np.ndarray) -> np.ndarray:
    """x / sqrt(mean(x^2) + eps) * gain (model.py:278-280)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + RMS_EPS) * gain


def silu(x: np.ndarray) -> np.ndarray:
    """Overflow-free x * sigmoid(x) (model.py:283-290)."""
    neg = x < 0
    z = np.exp(np.where(neg, x, -x))  # exp of -|x|
    return np.where(neg, x * z / (1.0 + z), x / (1.0 + z))


def gated_mlp(x: np.ndarray, layer) -> np.ndarray:
    """(silu(x Wg) * (x Wu)) Wd, no biases (model.py:293-294)."""
    return (silu(x @ layer.w_gate) * (x @ layer.w_up)) @ layer.w_down


def prefix_attention(
    q: np.ndarray,
    keys: np.ndarray,
    values: np.ndarray,
    horizon: np.ndarray,
    want_probs: bool = False,
):
    """Softmax attention where query row t may see keys 0..horizon[t].

    q is (T, H, Dh); keys/values are (S, Hkv, Dh) with H a multiple of Hkv
    (query head h reads kv head h // (H/Hkv)).  Every mask on the hot path is
    a key prefix: the causal prompt mask with an injected prefix
    (model.py:352-360) and the recompute horizon (recompute.py:92-93).  The
    arithmetic is model.py:297-315: scaled logits, -inf outside the mask,
    max-shifted exp, zeroed outside the mask, normalised, times V.

    Returns (ctx (T, H, Dh), probs (H, T, S) or None).
    """
    t, h, dh = q.shape
    s_len, hkv, _ = keys.shape
    group = h // hkv
    horizon = np.asarray(horizon, dtype=np.int64)
    ctx = np.empty_like(q)
    probs = np.zeros((h, t, s_len), dtype=q.dtype) if want_probs else None
    rows = max(1, _ATTN_BYTES_BUDGET // max(1, h * s_len * q.itemsize * 3))
    key_idx = np.arange(s_len)
    scale = math.sqrt(dh)  # python float: keeps f32 inputs f32
    for r0 in range(0, t, rows):
        r1 = min(t, r0 + rows)
        allowed = key_idx[None, :] <= horizon[r0:r1, None]  # (rows, S)
        for g in range(hkv):
            qg = q[r0:r1, g * group : (g + 1) * group, :].transpose(1, 0, 2)  # (grp, rows, Dh)
            logits = np.matmul(qg, keys[:, g, :].T) / scale  # (grp, rows, S)
            logits = np.where(allowed[None], logits, -np.inf)
            e = np.exp(logits - logits.max(axis=-1, keepdims=True))
            e = np.where(allowed[None], e, 0.0)
            p = e / e.sum(axis=-1, keepdims=True)
            ctx[r0:r1, g * group : (g + 1) * group, :] = np.matmul(p, values[:, g, :]).transpose(1, 0, 2)
            if want_probs:
                probs[g * group : (g + 1) * group, r0:r1, :] = p
    return ctx, probs


# ---------------------------------------------------------------------------
# Decoder forward (model.py:379-462)
# ---------------------------------------------------------------------------


@dataclass
class ForwardOut:
    keys: List[np.ndarray]  # per layer (T, Hkv, Dh), rotated at the run's positions
    values: List[np.ndarray]
    hidden: List[np.ndarray]  # per layer (T, d) block outputs
    probs: Optional[np.ndarray] = None  # (H, T, P+T) at the capture layer
    logits: Optional[np.ndarray] = None  # (vocab,) of the last token


def decoder_forward(
    weights,
    token_ids,
    positions,
    prefix: Optional[Sequence[tuple]] = None,
    capture_layer: Optional[int] = None,
    stop_after_capture: bool = False,
    want_logits: bool = True,
) -> ForwardOut:
    """Pre-norm decoder over a token run with an optional injected KV prefix.

    Token t sees the whole prefix plus run tokens 0..t (model.py:352-360).
    Prefix keys are used exactly as given (model.py:438-440).  RoPE at the
    supplied positions for the run's q and k (model.py:436-437).  With
    ``stop_after_capture`` the layers above ``capture_layer`` are not run
    (their outputs cannot change the captured probabilities).
    """
    cfg = weights.config
    tok = np.asarray(token_ids, dtype=np.int64)
    pos = np.asarray(positions, dtype=np.int64)
    if tok.ndim != 1 or tok.size == 0 or pos.shape != tok.shape:
        raise OracleError("token_ids/positions must be matching nonempty 1-D arrays")
    if tok.min() < 0 or tok.max() >= cfg.vocab_size:
        raise OracleError("token id outside vocabulary")
    if pos.min() < 0 or pos.max() >= cfg.max_position:
        raise OracleError("position outside [0, max_position)")
    t = tok.size
    h_q, hkv, dh = cfg.n_heads, _kv_heads(cfg), cfg.d_head
    p = 0 if prefix is None else int(prefix[0][0].shape[0])
    horizon = p + np.arange(t)
    dt = _dtype(weights)
    hid = weights.embedding[tok].astype(dt, copy=True)
    out = ForwardOut(keys=[], values=[], hidden=[])
    for li, lw in enumerate(weights.layers):
        x = rms_norm(hid, lw.attn_norm)
        q = rope_rotate((x @ lw.wq).reshape(t, h_q, dh), pos, cfg.rope_base)
        k = rope_rotate((x @ lw.wk).reshape(t, hkv, dh), pos, cfg.rope_base)
        v = (x @ lw.wv).reshape(t, hkv, dh)
        if prefix is not None:
            all_k = np.concatenate([prefix[li][0].astype(dt, copy=False), k], axis=0)
            all_v = np.concatenate([prefix[li][1].astype(dt, copy=False), v], axis=0)
        else:
            all_k, all_v = k, v
        capture = capture_layer is not None and li == capture_layer
        ctx, probs = prefix_attention(q, all_k, all_v, horizon, want_probs=capture)
        out.keys.append(k)
        out.values.append(v)
        if capture:
            out.probs = probs
            if stop_after_capture:
                return out
        hid = hid + ctx.reshape(t, cfg.d_model) @ lw.wo
        hid = hid + gated_mlp(rms_norm(hid, lw.mlp_norm), lw)
        out.hidden.append(hid.copy())
    if want_logits:
        out.logits = rms_norm(hid, weights.final_norm)[-1] @ weights.out_head
    return out


# ---------------------------------------------------------------------------
# Positions (positions.py:111-168)
# ---------------------------------------------------------------------------


def parse_mode(name) -> str:
    """Case-insensitive, '-' or '_' separated (positions.py:38-48)."""
    if hasattr(name, "value"):
        name = name.value
    key = str(name).strip().upper().replace("_", "-")
    if key not in GEOMETRY_MODES:
        raise OracleError(f"unknown geometry mode {name!r}")
    return key


def assign_positions(mode, chunk_lengths, prompt_length, prompt_offset=None, max_position=None):
    """Per-chunk context positions and prompt positions for a geometry.

    GLOBAL: chunks at their concatenated offsets, prompt after the context.
    HL-HP: chunks local, prompt after the longest chunk.  HL-TP: chunks local,
    prompt at prompt_offset (default sum of lengths).  TL-TP: chunks packed so
    the context ends right before the prompt (positions.py:131-158).
    """
    mode = parse_mode(mode)
    lens = [int(n) for n in chunk_lengths]
    if any(n < 1 for n in lens):
        raise OracleError("chunk lengths must all be >= 1")
    total = sum(lens)
    anchor = total if prompt_offset is None else int(prompt_offset)
    if mode == "GLOBAL":
        starts = list(np.cumsum([0] + lens[:-1])) if lens else []
        p0 = total
    elif mode == "HL-HP":
        starts = [0] * len(lens)
        p0 = max(lens) if lens else 0
    elif mode == "HL-TP":
        starts = [0] * len(lens)
        p0 = anchor
    else:  # TL-TP
        p0 = anchor
        tail = np.cumsum(lens[::-1])[::-1] if lens else []
        starts = [p0 - int(s) for s in tail]
        if starts and starts[0] < 0:
            raise OracleError("TL-TP pack underflows")
    ctx = [int(s) + np.arange(n, dtype=np.int64) for s, n in zip(starts, lens)]
    prm = int(p0) + np.arange(int(prompt_length), dtype=np.int64)
    if max_position is not None:
        top = max([int(c[-1]) for c in ctx] + ([int(prm[-1])] if prm.size else [0]))
        if top >= max_position:
            raise OracleError(f"assigned position {top} overflows max_position {max_position}")
    return ctx, prm


# ---------------------------------------------------------------------------
# Caches (cache.py:37-450)
# ---------------------------------------------------------------------------


@dataclass
class Chunk:
    """One chunk's stored KV: keys/values (L, len, Hkv, Dh) (cache.py:37-71)."""

    chunk_id: str
    token_ids: np.ndarray
    keys: np.ndarray
    values: np.ndarray
    positions: np.ndarray
    provenance: int = PREFILLED_LOCAL

    @property
    def length(self) -> int:
        return int(self.token_ids.size)


@dataclass
class Assembled:
    """Concatenated per-layer KV in declared order (cache.py:216-256)."""

    chunk_ids: List[str]
    chunk_lengths: List[int]
    token_ids: np.ndarray
    keys: np.ndarray  # (L, N + M, Hkv, Dh)
    values: np.ndarray
    row_positions: np.ndarray
    provenance: np.ndarray
    chunk_index: np.ndarray
    local_index: np.ndarray
    prompt_length: int = 0

    @property
    def context_length(self) -> int:
        return int(self.token_ids.size - self.prompt_length)

    @property
    def n_layers(self) -> int:
        return int(self.keys.shape[0])


def prefill_chunk(weights, chunk_id: str, token_ids) -> Chunk:
    """Chunk-local prefill: positions 0..len-1, causal (cache.py:74-99)."""
    tok = np.asarray(token_ids, dtype=np.int64)
    if tok.size == 0:
        raise OracleError(f"chunk {chunk_id!r} is empty")
    out = decoder_forward(weights, tok, np.arange(tok.size), want_logits=False)
    return Chunk(chunk_id, tok.copy(), np.stack(out.keys), np.stack(out.values),
                 np.arange(tok.size, dtype=np.int64), PREFILLED_LOCAL)


def assemble(chunks: Sequence[Chunk], prompt=None) -> Assembled:
    """Concatenate chunk KVs (and an optional prompt KV) in order (cache.py:259-322).

    ``prompt`` is (token_ids, keys (L,M,Hkv,Dh), values, positions) or None.
    """
    if not chunks and prompt is None:
        raise OracleError("nothing to assemble")
    lens = [c.length for c in chunks]
    tok = [c.token_ids for c in chunks]
    pos = [c.positions for c in chunks]
    prov = [np.full(c.length, c.provenance, np.uint8) for c in chunks]
    ks = [c.keys for c in chunks]
    vs = [c.values for c in chunks]
    m = 0
    if prompt is not None:
        ptok, pk, pv, ppos = prompt
        m = int(np.asarray(ptok).size)
        tok.append(np.asarray(ptok, np.int64))
        pos.append(np.asarray(ppos, np.int64))
        prov.append(np.full(m, FULL_PREFILL, np.uint8))
        ks.append(pk)
        vs.append(pv)
    cidx = [np.full(n, i, np.int64) for i, n in enumerate(lens)]
    lidx = [np.arange(n, dtype=np.int64) for n in lens]
    cat = lambda parts, dt: np.concatenate(parts) if parts else np.zeros(0, dt)  # noqa: E731
    return Assembled(
        chunk_ids=[c.chunk_id for c in chunks],
        chunk_lengths=lens,
        token_ids=cat(tok, np.int64),
        keys=np.concatenate(ks, axis=1),
        values=np.concatenate(vs, axis=1),
        row_positions=cat(pos, np.int64),
        provenance=cat(prov, np.uint8),
        chunk_index=cat(cidx, np.int64),
        local_index=cat(lidx, np.int64),
        prompt_length=m,
    )


def replace_rows(cache: Assembled, idx, new_keys, new_values, positions=None) -> Assembled:
    """Copy the cache, overwrite the listed context rows in every layer,
    record their rotation positions and RECOMPUTED_GLOBAL provenance
    (cache.py:325-374).  new_keys/new_values are (L, k, Hkv, Dh)."""
    idx = np.asarray(idx, dtype=np.int64).ravel()
    if idx.size == 0:
        return cache
    n = cache.context_length
    if idx.min() < 0 or idx.max() >= n:
        raise OracleError("replacement index outside context")
    if np.unique(idx).size != idx.size:
        raise OracleError("duplicate replacement indices")
    pos = idx.copy() if positions is None else np.asarray(positions, np.int64).ravel()
    keys, values = cache.keys.copy(), cache.values.copy()
    keys[:, idx] = new_keys
    values[:, idx] = new_values
    rp, pv = cache.row_positions.copy(), cache.provenance.copy()
    rp[idx] = pos
    pv[idx] = RECOMPUTED_GLOBAL
    return Assembled(cache.chunk_ids, cache.chunk_lengths, cache.token_ids, keys, values,
                     rp, pv, cache.chunk_index, cache.local_index, cache.prompt_length)


def decode_targets(cache: Assembled) -> np.ndarray:
    """Global decode layout: context row i at position i, prompt rows as stored."""
    n = cache.context_length
    return np.concatenate([np.arange(n, dtype=np.int64), cache.row_positions[n:]])


def decode_view(cache: Assembled, rope_base: float):
    """Keys of every row re-rotated to the decode layout; rows already there are
    copied bit-exactly (cache.py:382-403).  Returns (keys, values) (L, T, Hkv, Dh)."""
    delta = decode_targets(cache) - cache.row_positions
    moved = np.nonzero(delta != 0)[0]
    keys = cache.keys.copy()
    for li in range(cache.n_layers):
        if moved.size:
            keys[li, moved] = rope_rotate(cache.keys[li, moved], delta[moved], rope_base)
    return keys, cache.values


def full_prefill(weights, token_ids) -> Assembled:
    """Whole context prefilled at global positions (cache.py:406-425)."""
    tok = np.asarray(token_ids, dtype=np.int64)
    out = decoder_forward(weights, tok, np.arange(tok.size), want_logits=False)
    chunk = Chunk("full", tok, np.stack(out.keys), np.stack(out.values),
                  np.arange(tok.size, dtype=np.int64), FULL_PREFILL)
    return assemble([chunk])


def fidelity(a: Assembled, b: Assembled, rope_base: float):
    """(Frobenius, max-abs) distance of the decode views' context rows (cache.py:434-450)."""
    n = a.context_length
    ka, va = decode_view(a, rope_base)
    kb, vb = decode_view(b, rope_base)
    dk = ka[:, :n] - kb[:, :n]
    dv = va[:, :n] - vb[:, :n]
    fro = float(np.sqrt(np.sum(dk * dk) + np.sum(dv * dv)))
    worst = float(max(np.max(np.abs(dk)), np.max(np.abs(dv)))) if n else 0.0
    return fro, worst


# ---------------------------------------------------------------------------
# Attention-norm selection (selection.py:48-183, 263-300)
# ---------------------------------------------------------------------------


def default_norm_layer(n_layers: int) -> int:
    """min(L-1, floor(0.6 L)) (selection.py:48-50)."""
    return min(n_layers - 1, int(math.floor(0.6 * n_layers)))


def resolve_budget(n_context: int, ratio=None, topk=None) -> int:
    """ceil(ratio * N) or topk; must not exceed N (selection.py:83-87)."""
    if (ratio is None) == (topk is None):
        raise OracleError("exactly one of topk or ratio must be set")
    k = int(topk) if topk is not None else math.ceil(ratio * n_context)
    if k > n_context:
        raise OracleError(f"budget {k} exceeds context length {n_context}")
    return k


def column_scores(probs: np.ndarray, n_context: int) -> np.ndarray:
    """Head-mean, then sum over prompt rows of the context columns
    (selection.py:108-124).  probs is (H, M, S) or (M, S)."""
    a = np.asarray(probs, dtype=np.float64)
    if a.ndim == 3:
        a = a.mean(axis=0)
    if a.ndim != 2 or n_context > a.shape[1]:
        raise OracleError("bad attention shape for scoring")
    return a[:, :n_context].sum(axis=0)


def score_attention_norm(weights, cache: Assembled, prompt_ids, ctx_positions, prompt_positions,
                         norm_layer: int) -> np.ndarray:
    """Attention mass each context token receives from the prompt at
    ``norm_layer`` (selection.py:127-169): stored keys moved to the geometry's
    positions by rotation delta, prompt run forward on top, probabilities
    captured, head-mean, row-sum over context columns."""
    cfg = weights.config
    if not 0 <= norm_layer < cfg.n_layers:
        raise OracleError(f"norm_layer {norm_layer} outside [0, {cfg.n_layers})")
    n = cache.context_length
    target = np.asarray(ctx_positions, dtype=np.int64)
    if target.size != n:
        raise OracleError("position assignment does not cover the context")
    delta = target - cache.row_positions[:n]
    prefix = []
    for li in range(norm_layer + 1):
        k = cache.keys[li, :n]
        if np.any(delta != 0):
            k = rope_rotate(k, delta, cfg.rope_base)
        prefix.append((k, cache.values[li, :n]))
    prefix += [(cache.keys[li, :n], cache.values[li, :n]) for li in range(norm_layer + 1, cfg.n_layers)]
    out = decoder_forward(weights, prompt_ids, prompt_positions, prefix=prefix,
                          capture_layer=norm_layer, stop_after_capture=True, want_logits=False)
    return column_scores(out.probs, n)


def select_topk(scores, k: int) -> np.ndarray:
    """The k best indices by (score desc, index asc), returned ascending
    (selection.py:172-183)."""
    s = np.asarray(scores)
    if k < 0 or k > s.size:
        raise OracleError(f"k={k} outside [0, {s.size}]")
    if k == 0:
        return np.zeros(0, np.int64)
    order = np.lexsort((np.arange(s.size), -s))  # primary key last: score desc, then index
    return np.sort(order[:k]).astype(np.int64)


def score_cacheblend(weights, chunk_token_ids: Sequence, early_layers: int) -> np.ndarray:
    """CacheBlend baseline (selection.py:190-223): per token, the Euclidean
    distance between its block outputs in the chunk-local runs (positions
    0..len-1, causal within the chunk) and in one full-context causal run,
    summed over the first ``early_layers`` layers."""
    cfg = weights.config
    if early_layers < 1 or early_layers > cfg.n_layers:
        raise OracleError(f"early_layers {early_layers} outside [1, {cfg.n_layers}]")
    if not len(chunk_token_ids):
        raise OracleError("no chunks to score")
    local = [decoder_forward(weights, t, np.arange(len(t)), want_logits=False).hidden for t in chunk_token_ids]
    full_tok = np.concatenate([np.asarray(t, np.int64) for t in chunk_token_ids])
    full = decoder_forward(weights, full_tok, np.arange(full_tok.size), want_logits=False).hidden
    scores = np.zeros(full_tok.size, np.float64)
    for li in range(early_layers):
        loc = np.concatenate([h[li] for h in local], axis=0)
        scores += np.linalg.norm(loc - full[li], axis=1)
    return scores


def run_selection(weights, cache: Assembled, prompt_ids, ratio=None, topk=None, mode="GLOBAL",
                  norm_layer=None, prompt_offset=None):
    """Attention-norm strategy dispatch (selection.py:263-300).
    Returns (scores, selected)."""
    cfg = weights.config
    prompt_ids = np.asarray(prompt_ids, dtype=np.int64)
    ctx, prm = assign_positions(mode, cache.chunk_lengths, prompt_ids.size, prompt_offset,
                                cfg.max_position)
    nl = default_norm_layer(cfg.n_layers) if norm_layer is None else int(norm_layer)
    ctx_pos = np.concatenate(ctx) if ctx else np.zeros(0, np.int64)
    scores = score_attention_norm(weights, cache, prompt_ids, ctx_pos, prm, nl)
    k = resolve_budget(cache.context_length, ratio=ratio, topk=topk)
    return scores, select_topk(scores, k)


# ---------------------------------------------------------------------------
# Selective recomputation (recompute.py:56-122)
# ---------------------------------------------------------------------------


def make_plan(n_context: int, selected):
    """Sorted, unique, in-range selection; positions and causal horizons are
    the indices themselves (recompute.py:56-64)."""
    sel = np.sort(np.asarray(selected, dtype=np.int64).ravel())
    if sel.size and (sel[0] < 0 or sel[-1] >= n_context):
        raise OracleError("selected index outside context")
    if np.unique(sel).size != sel.size:
        raise OracleError("selected indices contain duplicates")
    return sel, sel.copy(), sel.copy()


def recompute_selected(weights, cache: Assembled, selected, positions=None, allowed_upto=None) -> Assembled:
    """Recompute the selected rows from their embeddings through every layer
    under the global causal mask and replace them (recompute.py:67-122).

    Per layer: fresh q/k/v of the selected tokens at their global positions;
    the layer's keys moved to the global layout (rows already there kept);
    fresh rows written over their slots so later selected tokens see them;
    prefix attention with horizon = allowed_upto; residual O-proj and MLP.
    """
    cfg = weights.config
    sel = np.asarray(selected, dtype=np.int64)
    if sel.size == 0:
        return cache
    n = cache.context_length
    pos = sel.copy() if positions is None else np.asarray(positions, np.int64)
    upto = sel.copy() if allowed_upto is None else np.asarray(allowed_upto, np.int64)
    if sel.min() < 0 or sel.max() >= n or np.any(upto >= n) or np.any(upto < sel):
        raise OracleError("invalid recompute plan")
    s = sel.size
    h_q, hkv, dh = cfg.n_heads, _kv_heads(cfg), cfg.d_head
    delta = np.arange(n, dtype=np.int64) - cache.row_positions[:n]
    moved = np.nonzero(delta != 0)[0]
    dt = _dtype(weights)
    hid = weights.embedding[cache.token_ids[sel]].astype(dt, copy=True)
    new_k = np.empty((cfg.n_layers, s, hkv, dh), dtype=cache.keys.dtype)
    new_v = np.empty_like(new_k)
    for li, lw in enumerate(weights.layers):
        x = rms_norm(hid, lw.attn_norm)
        k = rope_rotate((x @ lw.wk).reshape(s, hkv, dh), pos, cfg.rope_base)
        v = (x @ lw.wv).reshape(s, hkv, dh)
        new_k[li], new_v[li] = k, v
        if li == cfg.n_layers - 1:
            break  # the last layer's attention/MLP cannot change any K/V
        q = rope_rotate((x @ lw.wq).reshape(s, h_q, dh), pos, cfg.rope_base)
        keys = cache.keys[li, :n].copy()
        if moved.size:
            keys[moved] = rope_rotate(keys[moved], delta[moved], cfg.rope_base)
        keys[sel] = k
        values = cache.values[li, :n].copy()
        values[sel] = v
        ctx, _ = prefix_attention(q, keys, values, upto)
        hid = hid + ctx.reshape(s, cfg.d_model) @ lw.wo
        hid = hid + gated_mlp(rms_norm(hid, lw.mlp_norm), lw)
    return replace_rows(cache, sel, new_k, new_v, positions=pos)


# ---------------------------------------------------------------------------
# Information-flow chunk reordering (reorder.py:45-181)
# ---------------------------------------------------------------------------


def aggregate(values: np.ndarray, mode: str) -> float:
    """sum / mean / max of the selected first-pass scores; 0 if none (reorder.py:45-54)."""
    if mode not in CHUNK_SCORE_MODES:
        raise OracleError(f"unknown chunk score mode {mode!r}")
    if values.size == 0:
        return 0.0
    return float({"sum": np.sum, "mean": np.mean, "max": np.max}[mode](values))


def chunk_importance(weights, chunks: Sequence[Chunk], prompt_ids, budget: int, norm_layer=None,
                     chunk_score="sum"):
    """First pass: every chunk scored alone under HL-TP (chunk local, prompt at
    the sum of all lengths) with a per-chunk budget ceil(budget/K)
    (reorder.py:57-113).  Returns (importances, [(scores, selected)])."""
    if not chunks:
        raise OracleError("no chunks to score")
    if chunk_score not in CHUNK_SCORE_MODES:
        raise OracleError(f"unknown chunk score mode {chunk_score!r}")
    cfg = weights.config
    prompt_ids = np.asarray(prompt_ids, dtype=np.int64)
    nl = default_norm_layer(cfg.n_layers) if norm_layer is None else int(norm_layer)
    total = sum(c.length for c in chunks)
    per = math.ceil(budget / len(chunks)) if budget > 0 else 0
    imps = np.zeros(len(chunks), np.float64)
    passes = []
    for ci, c in enumerate(chunks):
        one = assemble([c])
        ctx, prm = assign_positions("HL-TP", [c.length], prompt_ids.size, total, cfg.max_position)
        sc = score_attention_norm(weights, one, prompt_ids, ctx[0], prm, nl)
        sel = select_topk(sc, min(per, c.length))
        imps[ci] = aggregate(sc[sel], chunk_score)
        passes.append((sc, sel))
    return imps, passes


def reorder_and_reselect(weights, chunks: Sequence[Chunk], prompt_ids, budget: int, norm_layer=None,
                         chunk_score="sum", sequential_input=False):
    """Stable ascending argsort of importances (most important chunk last,
    next to the prompt), re-assembly in that order, GLOBAL second pass with
    budget min(budget, N) (reorder.py:116-181).
    Returns (permutation, importances, cache, scores, selected)."""
    if sequential_input:
        raise OracleError("reorder requested on sequentially structured input")
    imps, _ = chunk_importance(weights, chunks, prompt_ids, budget, norm_layer, chunk_score)
    perm = np.argsort(imps, kind="stable").astype(np.int64)
    cache = assemble([chunks[i] for i in perm])
    cfg = weights.config
    nl = default_norm_layer(cfg.n_layers) if norm_layer is None else int(norm_layer)
    ctx, prm = assign_positions("GLOBAL", cache.chunk_lengths, np.asarray(prompt_ids).size, None,
                                cfg.max_position)
    scores = score_attention_norm(weights, cache, prompt_ids, np.concatenate(ctx), prm, nl)
    selected = select_topk(scores, min(budget, cache.context_length))
    return perm, imps, cache, scores, selected


# ---------------------------------------------------------------------------
# Convenience: the timed path as one call (harness.py:449-456)
# ---------------------------------------------------------------------------


def assemble_select_recompute(weights, chunks: Sequence[Chunk], prompt_ids, ratio=0.15, mode="GLOBAL",
                              norm_layer=None):
    """assemble -> run_selection -> make_plan -> recompute_selected."""
    cache = assemble(chunks)
    scores, sel = run_selection(weights, cache, prompt_ids, ratio=ratio, mode=mode, norm_layer=norm_layer)
    sel, pos, upto = make_plan(cache.context_length, sel)
    return recompute_selected(weights, cache, sel, pos, upto), scores, sel
