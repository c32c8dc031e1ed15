"""Property tests (hypothesis) of the host-side planning the kernels rely on:
rotation-delta tables, constant-delta runs, scorer work items and the
cross-rank top-k merge rule."""

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle as O
from paper_2603_05353_b200 import engine as E
from paper_2603_05353_b200 import sharding as SH
from paper_2603_05353_b200.cache import _delta_rows

deltas_st = st.lists(st.tuples(st.integers(-3, 3), st.integers(1, 6)), min_size=0, max_size=12).map(
    lambda runs: np.concatenate([np.full(n, d * 512, np.int64) for d, n in runs]) if runs else np.zeros(0, np.int64))


@settings(max_examples=200, deadline=None)
@given(deltas_st)
def test_delta_rows_maps_every_row_to_its_delta(deltas):
    tab, uniq = _delta_rows(deltas)
    assert tab.shape == deltas.shape and tab.dtype == np.int32
    assert np.all((tab >= 0) == (deltas != 0))
    assert np.array_equal(uniq[tab[tab >= 0]], deltas[deltas != 0])
    assert np.unique(uniq).size == uniq.size and np.all(uniq != 0)


@settings(max_examples=200, deadline=None)
@given(deltas_st, st.integers(0, 5))
def test_segments_are_maximal_constant_runs(deltas, offset):
    segs = E.segments_from_deltas(deltas, offset)
    rebuilt = np.concatenate([np.full(n, d, np.int64) for _, n, d in segs]) if segs else np.zeros(0, np.int64)
    assert np.array_equal(rebuilt, deltas)
    assert all(a[2] != b[2] for a, b in zip(segs, segs[1:]))  # maximal
    rows = [r for r, _, _ in segs]
    assert rows == sorted(rows) and (not segs or rows[0] == offset)


@settings(max_examples=100, deadline=None)
@given(st.lists(st.integers(1, 8192), min_size=1, max_size=64), st.sampled_from([1, 2, 4, 8]))
def test_tc_item_keys_is_a_block_multiple(run_lengths, hkv):
    g = E.PromptGroup(np.zeros(32, np.int64), np.arange(32), [(0, n, 1) for n in run_lengths])
    k = E._tc_item_keys([g], hkv, 4, 32)
    assert k % 128 == 0 and 128 <= k <= 2048


@settings(max_examples=150, deadline=None)
@given(st.integers(1, 60), st.integers(1, 4), st.data())
def test_merge_topk_equals_global_topk(n, world, data):
    vals = data.draw(st.lists(st.sampled_from([0.0, -0.0, 0.1, 0.25, 0.5, 1.5]), min_size=n, max_size=n))
    k = data.draw(st.integers(0, n))
    s = np.asarray(vals, np.float32)
    owner = np.asarray(data.draw(st.lists(st.integers(0, world - 1), min_size=n, max_size=n)))
    scores, idx = [], []
    for r in range(world):
        rows = np.flatnonzero(owner == r)
        loc = s[rows]
        kl = min(k, rows.size)
        order = sorted(range(rows.size), key=lambda i: (-float(loc[i]), int(rows[i])))[:kl]
        scores.append(torch.as_tensor(loc[order]))
        idx.append(torch.as_tensor(rows[order]))
    got = SH.merge_topk(scores, idx, k).numpy()
    want = O.select_topk(s.astype(np.float64), k)
    assert np.array_equal(got, want)


def test_selection_assert_helper_near_ties_only():
    """tests/helpers.assert_same_selection: exact when certified, near-tie
    swaps inside the error band tolerated, anything else rejected."""
    import pytest as _pt

    from helpers import assert_same_selection

    ref = np.array([5.0, 4.0, 3.0 + 1e-9, 3.0, 1.0])
    sel = np.array([0, 1, 2])
    assert assert_same_selection(sel, ref, ref, 3) == 0  # no error: certified
    got = ref.copy()
    got[3] += 2e-9  # index 3 now beats index 2: a near-tie within the error
    assert assert_same_selection(np.array([0, 1, 3]), got, ref, 3) == 1
    with _pt.raises(AssertionError):  # a token far outside the band
        assert_same_selection(np.array([0, 1, 4]), got, ref, 3)


def test_permutation_assert_helper_near_ties_only():
    import pytest as _pt

    from helpers import assert_same_permutation

    ref_imps = np.array([3.0, 1.0, 2.0, 2.0 + 1e-9])
    ref = np.argsort(ref_imps, kind="stable")  # [1, 2, 3, 0]
    got_imps = ref_imps.copy()
    got_imps[2] += 2e-9  # chunk 2 now sorts after chunk 3
    assert assert_same_permutation(np.argsort(got_imps, kind="stable"), ref, ref_imps, got_imps) == 2
    with _pt.raises(AssertionError):
        assert_same_permutation(np.array([2, 1, 3, 0]), ref, ref_imps, got_imps)
