"""Test helpers: convert device objects into oracle inputs (float64 copies of
the exact device values) and build small device scenarios."""

import numpy as np

import oracle as O


def to_np(t):
    return t.detach().double().cpu().numpy()


def oracle_chunk(ckv):
    return O.Chunk(ckv.chunk_id, ckv.token_ids.copy(), to_np(ckv.keys), to_np(ckv.values),
                   ckv.prefill_positions.copy(), int(ckv.provenance))


def oracle_cache(cache):
    return O.Assembled(list(cache.chunk_ids), list(cache.chunk_lengths), cache.token_ids.copy(), to_np(cache.keys),
                       to_np(cache.values), cache.row_positions.copy(), cache.provenance.copy(),
                       cache.chunk_index.copy(), cache.local_index.copy(), cache.prompt_length)


def rel_err(a, b):
    """max |a - b| / max |b| (norm-relative; elementwise rtol is meaningless
    for entries near zero)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def bf16_slab_tol(ref):
    """Tolerance for bf16-stored results: rtol 1e-2 of the tensor's scale
    (north star: scores and recomputed KV within rtol 1e-2 in bf16)."""
    return 1e-2
