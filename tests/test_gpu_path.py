"""End-to-end parity of the GPU path against the oracle on identical inputs.

Inputs: identical weights (device bf16 values, the oracle gets exact float64
copies) and the GPU's own chunk KVs (the path's input boundary: precomputed
chunk caches).  Bars (north star): selected index sets and reorder
permutations bit-exact; scores and recomputed KV within rtol 1e-2 (bf16) /
1e-4 (fp32 mode), measured as max|a-b| / max|b| per tensor."""

import numpy as np
import pytest

import oracle as O
from helpers import oracle_cache, oracle_chunk, rel_err, to_np

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2603_05353_b200 as P

    return P


def _setup(cfg, seed_w, precision, task, task_seed, host_weights=None):
    P = _pkg()
    hw = host_weights if host_weights is not None else P.init_weights(cfg, seed_w)
    dw = P.DeviceWeights.from_host(hw, precision)
    ow = dw.to_host()
    g = P.generate_task(task, task_seed) if task is not None else None
    return dw, ow, g


C1_TASK = dict(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32, vocab_size=1024)


@pytest.fixture(scope="module", params=[0, 1])
def c1(request, cuda):
    P = _pkg()
    dw, ow, g = _setup(P.c1_config(), 7, "bf16", P.SyntheticTask(**C1_TASK), request.param)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    return dw, ow, g, kvs


def test_c1_prefill_matches_oracle(c1):
    dw, ow, g, kvs = c1
    for ckv, spec in zip(kvs[:2], g.chunks[:2]):
        want = O.prefill_chunk(ow, spec.chunk_id, spec.token_ids)
        assert rel_err(to_np(ckv.keys), want.keys) <= 1e-2
        assert rel_err(to_np(ckv.values), want.values) <= 1e-2


def test_c1_selection_bit_exact(c1):
    P = _pkg()
    dw, ow, g, kvs = c1
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
    assert np.all(scores > 0)  # strictly positive: elementwise rtol is meaningful (north star: 1e-4 fp32-accurate)
    np.testing.assert_allclose(res.scores_numpy(), scores, rtol=1e-4, atol=0)
    np.testing.assert_array_equal(res.selected_numpy(), sel)
    assert res.budget == 308


def test_c1_recompute_matches_oracle(c1):
    P = _pkg()
    dw, ow, g, kvs = c1
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    sel = res.selected_numpy()
    want = O.recompute_selected(ow, oc, *O.make_plan(oc.context_length, sel))
    wk, wv = O.decode_view(want, dw.config.rope_base)
    before_k, _ = P.decode_view(cache, dw.config.rope_base)
    before_k = before_k.clone()
    out = P.recompute_selected(dw, cache, P.make_plan(cache, res.selected))
    gk, gv = P.decode_view(out, dw.config.rope_base)
    assert rel_err(to_np(gk), wk) <= 1e-2
    assert rel_err(to_np(gv), wv) <= 1e-2
    keep = np.setdiff1d(np.arange(cache.context_length), sel)
    assert to_np(gk)[:, keep].tobytes() == to_np(before_k)[:, keep].tobytes()
    assert (out.provenance[sel] == int(P.Provenance.RECOMPUTED_GLOBAL)).all()
    assert np.array_equal(out.row_positions[:cache.context_length], np.arange(cache.context_length))


def test_c1_reorder_bit_exact(c1):
    P = _pkg()
    dw, ow, g, kvs = c1
    plan, cache, second = P.reorder_and_reselect(dw, g.chunks, g.prompt_token_ids, budget=308, prefilled=kvs)
    perm, imps, _, scores, sel = O.reorder_and_reselect(ow, [oracle_chunk(c) for c in kvs], g.prompt_token_ids, 308)
    np.testing.assert_array_equal(plan.permutation, perm)
    np.testing.assert_allclose(plan.chunk_importance, imps, rtol=1e-4)
    np.testing.assert_array_equal(second.selected_numpy(), sel)
    np.testing.assert_allclose(second.scores_numpy(), scores, rtol=1e-4, atol=0)


def test_long_prompt_over_128_tokens_matches_oracle(cuda):
    """A 200-token prompt (the causal prompt keys span two 128-key items):
    selection bit-exact against the oracle."""
    P = _pkg()
    task = P.SyntheticTask(kind="uniform_noise", total_length=1024, fixed_size=256, prompt_length=32,
                           vocab_size=1024)
    dw, ow, g = _setup(P.c1_config(), 7, "bf16", task, 3)
    prompt = np.random.default_rng(3).integers(0, 1024, size=200)  # (the task generator caps prompts at its band)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, prompt, P.SelectionConfig(ratio=0.15))
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, prompt, ratio=0.15)
    np.testing.assert_allclose(res.scores_numpy(), scores, rtol=1e-4, atol=0)
    np.testing.assert_array_equal(res.selected_numpy(), sel)


# ---------------------------------------------------------------------------
# fp32 mode: the reference's tiny configs, 1e-4 bars
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def tiny(cuda):
    P = _pkg()
    cfg = P.ModelConfig(n_layers=2, n_heads=2, d_model=16, d_head=8, d_ff=32, vocab_size=64, max_position=4096)
    dw, ow, _ = _setup(cfg, 7, "f32", None, None)
    return P, cfg, dw, ow


def test_fp32_golden_direct(tiny, golden_small):
    """Reference outputs (golden) reproduced from the reference's own chunk KVs."""
    P, cfg, dw, ow = tiny
    import torch

    toks, prompt = golden_small["tiny_tokens"], golden_small["tiny_prompt"]
    chunks = P.make_chunks(toks, [8, 8, 8])
    kvs = [P.cache.chunk_from_host(f"c{i}", toks[8 * i:8 * i + 8], golden_small["tiny_chunk_keys"][i],
                                   golden_small["tiny_chunk_values"][i], np.arange(8), 0, dw.fingerprint(),
                                   torch.float32) for i in range(3)]
    cache = P.assemble(kvs)
    for mode, off in (("GLOBAL", None), ("HL-HP", None), ("HL-TP", 200), ("TL-TP", 200)):
        geo = P.GeometryConfig(mode=mode, prompt_length=4, chunk_lengths=(8, 8, 8), prompt_offset=off)
        s = P.score_attention_norm(dw, cache, prompt, P.assign_positions(geo, chunks), 1)
        want = golden_small[f"tiny_scores_{mode}"]
        assert rel_err(s.double().cpu().numpy(), want) <= 1e-5
        np.testing.assert_array_equal(P.select_topk(s, 6).cpu().numpy(), golden_small[f"tiny_sel6_{mode}"])
    out = P.recompute_selected(dw, P.assemble(kvs), P.make_plan(cache, np.array([3, 11, 20])))
    dk, dv = P.decode_view(out, cfg.rope_base)
    assert rel_err(to_np(dk), golden_small["tiny_rec_decode_keys"]) <= 1e-4
    assert rel_err(to_np(dv), golden_small["tiny_rec_values"]) <= 1e-4
    for budget in (1, 6, 12):
        plan, _, second = P.reorder_and_reselect(dw, chunks, prompt, budget=budget, prefilled=kvs)
        np.testing.assert_array_equal(plan.permutation, golden_small[f"tiny_reorder{budget}_perm"])
        np.testing.assert_array_equal(second.selected_numpy(), golden_small[f"tiny_reorder{budget}_sel"])


def test_fp32_full_recompute_equals_full_prefill(cuda):
    """Criterion 1 (test_acceptance.py:49-63): ratio 1.0 reproduces full prefill."""
    P = _pkg()
    cfg = P.toy_config()
    dw, ow, _ = _setup(cfg, 7, "f32", None, None)
    for seed in range(3):
        task = P.SyntheticTask(kind="uniform_noise", total_length=256, fixed_size=64, prompt_length=8)
        g = P.generate_task(task, seed)
        kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
        cache = P.assemble(kvs)
        ref = P.full_prefill(dw, cache.token_ids)
        res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids, P.SelectionConfig(ratio=1.0))
        out = P.recompute_selected(dw, cache, P.make_plan(cache, res.selected))
        assert P.cache_fidelity(out, ref, cfg.rope_base).max_abs <= 1e-4


def test_fp32_prefill_and_selection_vs_oracle(tiny):
    P, cfg, dw, ow = tiny
    rng = np.random.default_rng(21)
    toks = rng.integers(0, 64, 32)
    prompt = rng.integers(0, 64, 4)
    chunks = P.make_chunks(toks, [8, 8, 8, 8])
    kvs = [P.prefill_chunk(dw, c) for c in chunks]
    for ckv, spec in zip(kvs, chunks):
        want = O.prefill_chunk(ow, spec.chunk_id, spec.token_ids)
        assert rel_err(to_np(ckv.keys), want.keys) <= 1e-5
    cache = P.assemble(kvs)
    res = P.run_selection(dw, chunks, cache, prompt, P.SelectionConfig(topk=10))
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    s, sel = O.run_selection(ow, oc, prompt, topk=10)
    np.testing.assert_allclose(res.scores_numpy(), s, rtol=1e-5, atol=0)
    np.testing.assert_array_equal(res.selected_numpy(), sel)
    out = P.recompute_selected(dw, cache, P.make_plan(cache, res.selected))
    want = O.recompute_selected(ow, oc, *O.make_plan(32, sel))
    wk, wv = O.decode_view(want, cfg.rope_base)
    gk, gv = P.decode_view(out, cfg.rope_base)
    assert rel_err(to_np(gk), wk) <= 1e-4 and rel_err(to_np(gv), wv) <= 1e-4


def test_empty_plan_identity_and_validation(tiny):
    P, cfg, dw, ow = tiny
    chunks = P.make_chunks(np.arange(16) % 64, [8, 8])
    cache = P.assemble([P.prefill_chunk(dw, c) for c in chunks])
    assert P.recompute_selected(dw, cache, P.make_plan(cache, np.array([], np.int64))) is cache
    with pytest.raises(P.ConfigurationError):
        P.make_plan(cache, np.array([0, 0]))
    with pytest.raises(P.ConfigurationError):
        P.make_plan(cache, np.array([16]))
    with pytest.raises(P.ConfigurationError):
        P.select_topk(np.array([1.0]), 2)


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_gqa_path_vs_oracle(cuda, precision):
    P = _pkg()
    cfg = P.ModelConfig(n_layers=2, n_heads=4, d_model=64, d_head=16, d_ff=96, vocab_size=128, max_position=4096,
                        n_kv_heads=2)
    dw, ow, _ = _setup(cfg, 11, precision, None, None)
    rng = np.random.default_rng(3)
    toks, prompt = rng.integers(0, 128, 96), rng.integers(0, 128, 8)
    chunks = P.make_chunks(toks, [32, 32, 32])
    kvs = [P.prefill_chunk(dw, c) for c in chunks]
    cache = P.assemble(kvs)
    res = P.run_selection(dw, chunks, cache, prompt, P.SelectionConfig(ratio=0.2))
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    s, sel = O.run_selection(ow, oc, prompt, ratio=0.2)
    np.testing.assert_allclose(res.scores_numpy(), s, rtol=1e-4, atol=0)
    np.testing.assert_array_equal(res.selected_numpy(), sel)
    out = P.recompute_selected(dw, cache, P.make_plan(cache, res.selected))
    want = O.recompute_selected(ow, oc, *O.make_plan(96, sel))
    wk, wv = O.decode_view(want, cfg.rope_base)
    gk, gv = P.decode_view(out, cfg.rope_base)
    tol = 1e-2 if precision == "bf16" else 1e-4
    assert rel_err(to_np(gk), wk) <= tol and rel_err(to_np(gv), wv) <= tol


def test_tc_scorer_gqa_dh128_vs_simt_and_oracle(cuda):
    """tcgen05 scorer (G = 4 heads x 32 prompt rows = 128-row tiles, ragged
    192-row chunks -> partial key items) vs the SIMT scorer and the oracle."""
    P = _pkg()
    from paper_2603_05353_b200 import engine as E

    cfg = P.ModelConfig(n_layers=3, n_heads=8, d_model=1024, d_head=128, d_ff=512, vocab_size=256,
                        max_position=8192, n_kv_heads=2)
    dw, ow, _ = _setup(cfg, 5, "bf16", None, None)
    rng = np.random.default_rng(9)
    toks, prompt = rng.integers(0, 256, 768), rng.integers(0, 256, 32)
    chunks = P.make_chunks(toks, [192] * 4)
    kvs = [P.prefill_chunk(dw, c) for c in chunks]
    cache = P.assemble(kvs)
    geo = P.GeometryConfig(mode="global", prompt_length=32, chunk_lengths=(192,) * 4)
    a = P.assign_positions(geo, chunks)
    grp = E.PromptGroup(prompt, a.prompt_positions, E.segments_from_deltas(a.context_concat() - cache.row_positions))
    tc = E.prompt_forward(dw, cache.keys, cache.values, [grp], capture_layer=2).scores[:768].double().cpu().numpy()
    simt = E.prompt_forward(dw, cache.keys, cache.values, [grp], capture_layer=2,
                            impl="simt").scores[:768].double().cpu().numpy()
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    s, sel = O.run_selection(ow, oc, prompt, ratio=0.15, norm_layer=2)
    assert rel_err(tc, s) <= 1e-5 and rel_err(simt, s) <= 1e-5
    np.testing.assert_array_equal(P.select_topk(tc, sel.size).cpu().numpy(), sel)
    res = P.run_selection(dw, chunks, cache, prompt, P.SelectionConfig(ratio=0.15, norm_layer=2))
    np.testing.assert_array_equal(res.selected_numpy(), sel)


@pytest.mark.parametrize("precision", ["bf16", "f32"])
def test_first_token_over_recomputed_cache(cuda, precision):
    """Decode step over the recomputed cache (harness.py:458-469) vs the
    oracle's forward on the same cache (its decode view)."""
    P = _pkg()
    dw, ow, g = _setup(P.c1_config(), 7, precision, P.SyntheticTask(**C1_TASK), 0)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    cache = P.assemble(kvs)
    before = P.first_token_logits(dw, cache, g.prompt_token_ids)  # stale cache, decode view on the fly
    oc = oracle_cache(cache)
    dk, dv = O.decode_view(oc, dw.config.rope_base)
    n = oc.context_length
    want0 = O.decoder_forward(ow, g.prompt_token_ids, n + np.arange(32),
                              prefix=[(dk[l, :n], dv[l, :n]) for l in range(dk.shape[0])]).logits
    assert rel_err(before.double().cpu().numpy(), want0) <= 1e-4
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
    out = P.recompute_selected(dw, cache, P.make_plan(cache, res.selected))
    logits = P.first_token_logits(dw, out, g.prompt_token_ids)
    oc2 = oracle_cache(out)
    want = O.decoder_forward(ow, g.prompt_token_ids, n + np.arange(32),
                             prefix=[(oc2.keys[l, :n], oc2.values[l, :n]) for l in range(oc2.n_layers)]).logits
    assert rel_err(logits.double().cpu().numpy(), want) <= 1e-4
    assert P.greedy_token(logits) == int(np.argmax(want))


# ---------------------------------------------------------------------------
# CacheBlend baseline selector on the GPU (selection.py:190-223)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("early", [1, 2])
def test_fp32_cacheblend_vs_golden(tiny, golden_small, early):
    """fp32 mode against the reference's own scores (tiny config)."""
    P, _, dw, _ = tiny
    toks = golden_small["tiny_tokens"]
    chunks = [P.ChunkSpec(f"c{i}", toks[8 * i:8 * i + 8], i) for i in range(3)]
    s = P.score_cacheblend(dw, chunks, early).cpu().numpy()
    assert rel_err(s, golden_small[f"tiny_cacheblend{early}_scores"]) <= 1e-4
    if early == 2:
        cache = P.assemble([P.prefill_chunk(dw, c) for c in chunks])
        res = P.run_selection(dw, chunks, cache, golden_small["tiny_prompt"],
                              P.SelectionConfig(strategy="cacheblend", topk=6, cacheblend_layers=2))
        np.testing.assert_array_equal(res.selected_numpy(), golden_small["tiny_cacheblend_sel6"])


def test_c1_cacheblend_vs_oracle(c1):
    """BASELINE config 1, bf16 path, against the oracle on identical weights:
    scores within the bf16 bar; the selected sets overlap almost entirely
    (the bf16 hidden states move near-tied scores)."""
    P = _pkg()
    dw, ow, g, kvs = c1
    s = P.score_cacheblend(dw, g.chunks, 2).cpu().numpy()
    want = O.score_cacheblend(ow, [c.token_ids for c in g.chunks], 2)
    assert rel_err(s, want) <= 1e-2
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids,
                          P.SelectionConfig(strategy="cacheblend", ratio=0.15, cacheblend_layers=2))
    got = res.selected_numpy()
    ref = O.select_topk(want, 308)
    assert got.size == 308 and np.intersect1d(got, ref).size >= 0.95 * 308
    # the first chunk sits at its local positions in both runs: zero deviation
    np.testing.assert_array_equal(s[:256], np.zeros(256))


def test_c1_cacheblend_f32_set_bit_exact(cuda):
    """BASELINE config 1 in the fp32 mode: CacheBlend's deviation scores
    (fp64-accumulated on the GPU) against the oracle elementwise, and the
    selected set bit-exact (selection.py:191-225; the bf16 mode above only
    bounds the overlap because bf16 hidden states move near-tied scores)."""
    P = _pkg()
    dw, ow, g = _setup(P.c1_config(), 7, "f32", P.SyntheticTask(**C1_TASK), 0)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    s = P.score_cacheblend(dw, g.chunks, 2).cpu().numpy()
    want = O.score_cacheblend(ow, [c.token_ids for c in g.chunks], 2)
    pos = want > 0
    np.testing.assert_allclose(s[pos], want[pos], rtol=1e-4, atol=0)
    assert np.all(np.abs(s[~pos]) <= 1e-4 * want.max())  # the first chunk: zero in the oracle
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids,
                          P.SelectionConfig(strategy="cacheblend", ratio=0.15, cacheblend_layers=2))
    np.testing.assert_array_equal(res.selected_numpy(), O.select_topk(want, 308))


def test_cacheblend_validation(tiny):
    P, _, dw, _ = tiny
    chunks = [P.ChunkSpec("a", np.arange(5), 0)]
    with pytest.raises(P.ConfigurationError):
        P.score_cacheblend(dw, chunks, 0)
    with pytest.raises(P.ConfigurationError):
        P.score_cacheblend(dw, chunks, dw.config.n_layers + 1)
    with pytest.raises(P.ConfigurationError):
        P.score_cacheblend(dw, [], 1)
    s = P.score_cacheblend(dw, chunks, 2).cpu().numpy()
    np.testing.assert_array_equal(s, np.zeros(5))


# ---------------------------------------------------------------------------
# batched chunk prefill (cache.py:74-99 for many chunks in one layer stack)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("precision,cfg_name", [("bf16", "c1"), ("bf16", "gqa7"), ("f32", "c1")])
def test_prefill_chunks_matches_oracle_per_chunk(cuda, precision, cfg_name):
    """One block-diagonal layer stack over ragged chunks (lengths not multiples
    of the 32-token / 18-token attention tiles, a 1-token chunk) equals the
    oracle's per-chunk prefill, and the per-chunk GPU prefill."""
    P = _pkg()
    if cfg_name == "c1":
        cfg = P.c1_config()
    else:  # GQA group 7 (Qwen2.5-VL-like tiles of 18 tokens x 7 heads)
        cfg = P.ModelConfig(n_layers=2, n_heads=14, d_model=1792, d_head=128, d_ff=512, vocab_size=512,
                            max_position=8192, n_kv_heads=2)
    dw, ow, _ = _setup(cfg, 7, precision, None, 0)
    rng = np.random.default_rng(1)
    lens = [100, 37, 300, 1, 64, 256]
    chunks = [P.ChunkSpec(f"c{i}", rng.integers(0, cfg.vocab_size, size=n)) for i, n in enumerate(lens)]
    got = P.prefill_chunks(dw, chunks)
    tol = 1e-2 if precision == "bf16" else 1e-4
    for ckv, spec in zip(got, chunks):
        want = O.prefill_chunk(ow, spec.chunk_id, spec.token_ids)
        assert rel_err(to_np(ckv.keys), want.keys) <= tol
        assert rel_err(to_np(ckv.values), want.values) <= tol
        one = P.prefill_chunk(dw, spec)
        assert rel_err(to_np(ckv.keys), to_np(one.keys)) <= tol
        np.testing.assert_array_equal(ckv.prefill_positions, np.arange(spec.local_length))
    # the batched store feeds the path like separately prefilled chunks
    cache = P.assemble(got)
    assert cache.context_length == sum(lens)


def test_store_path_fuses_rotation_into_assembly(cuda):
    """Chunks from prefill_chunks take the fused path (scoring straight from
    the store, one rotating gather into the decode layout): the selected set
    and scores equal the two-pass path's bit for bit, the oracle's set, and the
    recomputed cache equals the two-pass path's; the rotating gather equals
    assemble + decode_view bit for bit."""
    P = _pkg()
    task = P.SyntheticTask(**C1_TASK)
    dw, ow, g = _setup(P.c1_config(), 7, "bf16", task, 0)
    kvs = P.prefill_chunks(dw, g.chunks)
    assert all(c.store is kvs[0].store for c in kvs)
    cfg = P.SelectionConfig(ratio=0.15)
    fused = P.assemble_select_recompute(dw, kvs, g.chunks, g.prompt_token_ids, cfg)
    plain_kvs = [P.ChunkKV(c.chunk_id, c.token_ids, c.keys.clone(), c.values.clone(), c.prefill_positions,
                           c.provenance, c.model_fingerprint) for c in kvs]  # no store: the two-pass path
    plain = P.assemble_select_recompute(dw, plain_kvs, g.chunks, g.prompt_token_ids, cfg)
    np.testing.assert_array_equal(fused.selection.selected_numpy(), plain.selection.selected_numpy())
    np.testing.assert_array_equal(fused.selection.scores_numpy(), plain.selection.scores_numpy())
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    _, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
    np.testing.assert_array_equal(fused.selection.selected_numpy(), sel)
    import torch

    assert torch.equal(fused.cache.keys, plain.cache.keys) and torch.equal(fused.cache.values, plain.cache.values)
    np.testing.assert_array_equal(fused.cache.row_positions, plain.cache.row_positions)
    from paper_2603_05353_b200.cache import assemble_decode_layout

    rot = assemble_decode_layout(kvs, dw.config.rope_base)
    want_k, _ = P.decode_view(P.assemble(kvs), dw.config.rope_base)
    assert torch.equal(rot.keys, want_k[:, :rot.context_length])
    np.testing.assert_array_equal(rot.row_positions, np.arange(rot.context_length))


def test_store_reorder_path_matches_plain_reorder(cuda):
    """The reorder over chunks of one store slab (the first pass reads every
    chunk's rows in place, no assembled copy) returns the path over separately
    prefilled chunks' permutation, importances, first- and second-pass scores
    and sets and recomputed cache bit for bit, and the oracle's permutation
    and second-pass set."""
    import torch

    P = _pkg()
    task = P.SyntheticTask(**C1_TASK)
    dw, ow, g = _setup(P.c1_config(), 7, "bf16", task, 0)
    kvs = P.prefill_chunks(dw, g.chunks)
    cfg = P.SelectionConfig(ratio=0.15)
    fused = P.assemble_select_recompute(dw, kvs, g.chunks, g.prompt_token_ids, cfg, reorder=True)
    plain_kvs = [P.ChunkKV(c.chunk_id, c.token_ids, c.keys.clone(), c.values.clone(), c.prefill_positions,
                           c.provenance, c.model_fingerprint) for c in kvs]  # no store: reorder_and_reselect
    plain = P.assemble_select_recompute(dw, plain_kvs, g.chunks, g.prompt_token_ids, cfg, reorder=True)
    fr, pr = fused.reorder, plain.reorder
    np.testing.assert_array_equal(fr.permutation, pr.permutation)
    np.testing.assert_array_equal(fr.chunk_importance, pr.chunk_importance)
    for a, b in zip(fr.first_pass, pr.first_pass):
        np.testing.assert_array_equal(a.scores_numpy(), b.scores_numpy())
        np.testing.assert_array_equal(a.selected_numpy(), b.selected_numpy())
    np.testing.assert_array_equal(fused.selection.scores_numpy(), plain.selection.scores_numpy())
    np.testing.assert_array_equal(fused.selection.selected_numpy(), plain.selection.selected_numpy())
    assert torch.equal(fused.cache.keys, plain.cache.keys) and torch.equal(fused.cache.values, plain.cache.values)
    np.testing.assert_array_equal(fused.cache.row_positions, plain.cache.row_positions)
    budget = cfg.resolve_budget(sum(c.local_length for c in g.chunks))
    perm, _, _, _, sel = O.reorder_and_reselect(ow, [oracle_chunk(c) for c in kvs], g.prompt_token_ids, budget)
    np.testing.assert_array_equal(fr.permutation, perm)
    np.testing.assert_array_equal(fused.selection.selected_numpy(), sel)


@pytest.mark.parametrize("ratio", [0.15, 0.05])
def test_query_graph_replays_match_eager(cuda, ratio):
    """The CUDA-graph replay of a whole query (QueryGraph: ~450 launches as
    one graph) returns the eager path's selected set, scores, recomputed slab
    and row metadata bit for bit, for several prompts replayed through one
    captured graph (the prompt ids reach it through a static device buffer);
    the C1 selection also equals the oracle's.  ratio 0.05 exercises the
    attention's key-split workspace (stream-ordered allocation inside the
    graph)."""
    import torch

    P = _pkg()
    task = P.SyntheticTask(**C1_TASK)
    dw, ow, g = _setup(P.c1_config(), 7, "bf16", task, 0)
    kvs = P.prefill_chunks(dw, g.chunks)
    cfg = P.SelectionConfig(ratio=ratio)
    rng = np.random.default_rng(5)
    prompts = [np.asarray(g.prompt_token_ids)] + [rng.integers(0, 1024, 32) for _ in range(2)]
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    for prompt in prompts + prompts[:1]:
        eager = P.assemble_select_recompute(dw, kvs, g.chunks, prompt, cfg)
        e_sel, e_sc = eager.selection.selected_numpy(), eager.selection.scores_numpy()
        e_k, e_v, e_rp = eager.cache.keys.clone(), eager.cache.values.clone(), eager.cache.row_positions.copy()
        del eager
        got = P.assemble_select_recompute(dw, kvs, g.chunks, prompt, cfg, graph=True)
        np.testing.assert_array_equal(got.selection.selected_numpy(), e_sel)
        np.testing.assert_array_equal(got.selection.scores_numpy(), e_sc)
        assert torch.equal(got.cache.keys, e_k) and torch.equal(got.cache.values, e_v)
        np.testing.assert_array_equal(got.cache.row_positions, e_rp)
        _, sel = O.run_selection(ow, oc, prompt, ratio=ratio)
        np.testing.assert_array_equal(got.selection.selected_numpy(), sel)
    qg = P.query_graph(dw, kvs, g.chunks, 32, cfg)
    assert qg.launches > 20  # the whole query is in the graph (C1: 2 layers)
    with pytest.raises(P.ConfigurationError):
        qg.run(np.zeros(31, np.int64))
    with pytest.raises(P.ConfigurationError):
        qg.run(np.full(32, 5000, np.int64))


def test_c1_fp64_selection_matches_oracle(c1):
    """score_precision='fp64' at BASELINE config 1: float64 scores to ~1e-12 of
    the oracle's, the same selected set; through run_selection and through the
    store path of assemble_select_recompute (exact.py)."""
    P = _pkg()
    dw, ow, g, kvs = c1
    cache = P.assemble(kvs)
    cfg64 = P.SelectionConfig(ratio=0.15, score_precision="fp64")
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids, cfg64)
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
    np.testing.assert_allclose(res.scores_numpy(), scores, rtol=1e-10, atol=0)
    np.testing.assert_array_equal(res.selected_numpy(), sel)
    store = P.prefill_chunks(dw, g.chunks)
    out = P.assemble_select_recompute(dw, store, g.chunks, g.prompt_token_ids, cfg64, graph=True)  # eager (fp64)
    np.testing.assert_array_equal(out.selection.selected_numpy(), sel)


def test_c1_fp64_reorder_matches_oracle(c1):
    P = _pkg()
    dw, ow, g, kvs = c1
    plan, cache, second = P.reorder_and_reselect(dw, g.chunks, g.prompt_token_ids, budget=308, prefilled=kvs,
                                                 score_precision="fp64")
    perm, imps, _, scores, sel = O.reorder_and_reselect(ow, [oracle_chunk(c) for c in kvs], g.prompt_token_ids, 308)
    np.testing.assert_allclose(plan.chunk_importance, imps, rtol=1e-10)
    np.testing.assert_array_equal(plan.permutation, perm)
    np.testing.assert_allclose(second.scores_numpy(), scores, rtol=1e-10, atol=0)
    np.testing.assert_array_equal(second.selected_numpy(), sel)
