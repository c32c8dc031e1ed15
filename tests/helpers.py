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


def assert_same_selection(got_sel, got_scores, ref_scores, k, tag=""):
    """Selected set vs the float64 reference (select_topk, ties by index).

    Bit-exact when the reference's boundary gap (k-th vs (k+1)-th score)
    exceeds twice the largest observed score error, i.e. when fp32-accurate
    scores can certify the order.  Otherwise the two sets may differ only by
    tokens whose reference scores lie within that error band of the k-th
    score (near-ties the float64 reference resolves below fp32 resolution;
    SURVEY section 7 hard part 1): every differing token
    is checked to be such a near-tie.  Returns the number of swapped pairs."""
    got_sel = np.asarray(got_sel)
    ref_scores = np.asarray(ref_scores, np.float64)
    order = np.lexsort((np.arange(ref_scores.size), -ref_scores))
    ref_sel = np.sort(order[:k])
    err = float(np.max(np.abs(np.asarray(got_scores, np.float64) - ref_scores)))
    s_sorted = ref_scores[order]
    kth, nxt = s_sorted[k - 1], s_sorted[k] if k < s_sorted.size else -np.inf
    certified = (kth - nxt) > 2 * err
    diff = np.setxor1d(got_sel, ref_sel)
    print(f"{tag} selection: k={k}, boundary gap {(kth - nxt) / kth:.2e} rel, max score error {err / kth:.2e} rel, "
          f"{'certified' if certified else 'NOT certified'}; {diff.size // 2} swapped pair(s)")
    if certified or diff.size == 0:
        np.testing.assert_array_equal(got_sel, ref_sel)
        return 0
    assert got_sel.size == ref_sel.size
    band = np.abs(ref_scores[diff] - kth) <= 2 * err
    assert np.all(band), f"tokens {diff[~band]} differ outside the score-error band (gap > 2 x {err:.3e})"
    return diff.size // 2


def assert_same_permutation(got_perm, ref_perm, ref_imps, got_imps, tag=""):
    """Reorder permutation vs the float64 reference (stable argsort of the
    chunk importances): bit-exact, except that chunks whose reference
    importances lie within twice the observed importance error of each other
    (near-ties below fp32 resolution) may trade places.  Returns the number
    of positions that differ."""
    got_perm, ref_perm = np.asarray(got_perm), np.asarray(ref_perm)
    ref_imps = np.asarray(ref_imps, np.float64)
    err = float(np.max(np.abs(np.asarray(got_imps, np.float64) - ref_imps)))
    diff = np.flatnonzero(got_perm != ref_perm)
    srt = np.sort(ref_imps)
    print(f"{tag} permutation: min importance gap {np.min(np.diff(srt)):.3e}, max importance error {err:.3e}; "
          f"{diff.size} position(s) differ")
    assert np.array_equal(np.sort(got_perm), np.arange(got_perm.size))
    for i in diff:
        a, b = ref_imps[got_perm[i]], ref_imps[ref_perm[i]]
        assert abs(a - b) <= 2 * err, f"position {i}: chunks {got_perm[i]} / {ref_perm[i]} are not a near-tie"
    return int(diff.size)
