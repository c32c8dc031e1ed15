"""Oracle parity at the BASELINE.json shapes (the north star's "identical
selected-token sets to the CPU reference" at Llama-3-8B width), reduced only
in depth so the float64 oracle finishes in test time.

Inputs are identical on both sides: the device's bf16 weights (the oracle gets
exact float64 copies) and the GPU's own chunk KVs (the path's input boundary,
cache.py:74-99), as SURVEY §7 hard part 1 prescribes.

* C2 width (d 4096, 32 q / 8 kv heads, d_ff 14336, vocab 128256, RoPE 5e5)
  over the real 32K context in 16 x 2048 chunks, 4 layers (norm layer 2):
  every score agrees to elementwise rtol 1e-4 (scores are strictly
  positive, so elementwise rtol is meaningful) and the selected set is
  bit-exact whenever the boundary gap exceeds twice the observed score
  error; below that the sets may differ only by near-tied tokens inside the
  error band, which is asserted token by token and printed
  (tests/helpers.py:assert_same_selection; selection.py:127-183,
  test_acceptance.py:191-202).
* C4 width (Qwen2.5-VL-7B LM: d 3584, 28 q / 4 kv heads -> GQA group 7,
  d_ff 18944), 24 x 1280 image-token chunks + 4 x 512 text chunks.
* C3: the information-flow reorder over 64 x 2048 chunks (128K context) at
  Llama-3-8B width, 2 layers: permutation and second-pass set bit-exact
  (reorder.py:116-181).
* depth: all 32 layers at C1 width (norm layer 19), selection bit-exact and
  the recomputed K/V rows of every layer against the float64 oracle
  (recompute.py:97-118).  bf16 recompute error grows with depth: the K/V rows
  are stored in bf16 (layer 0 is already ~4e-3 of the tensor's max from that
  rounding alone) and every layer rounds its four GEMM inputs to bf16, so the
  max-norm error climbs to ~1e-2 by layer 31 (printed per layer).  Bars: the
  Frobenius-relative error of every layer <= 1e-2 (the north star's bf16
  rtol, in the norm the reference's own cache_fidelity uses,
  cache.py:434-450) and the max-norm error <= 1.5e-2."""

import dataclasses
import math

import numpy as np
import pytest

import oracle as O
from helpers import assert_same_permutation, assert_same_selection, oracle_chunk, rel_err, to_np

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def oracle_weights(dw, n_layers):
    """Float64 copies of the device weights' first n_layers layers (the
    oracle's scoring pass stops at the capture layer; the output head is not
    needed)."""
    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200.model import LayerWeights, deinterleave_gu

    def hd(t):
        return t.detach().double().cpu().numpy()

    def ht(t):
        return np.ascontiguousarray(hd(t).T)

    c = dw.config
    layers = []
    for dl in dw.layers[:n_layers]:
        qkv = ht(dl.wqkv)
        g_t, u_t = deinterleave_gu(hd(dl.wgu), dw.gu_block)
        layers.append(LayerWeights(hd(dl.attn_norm), qkv[:, :c.d_model], qkv[:, c.d_model:c.d_model + c.kv_dim],
                                     qkv[:, c.d_model + c.kv_dim:], ht(dl.wo), hd(dl.mlp_norm),
                                     np.ascontiguousarray(g_t.T), np.ascontiguousarray(u_t.T), ht(dl.wdown)))
    return P.Weights(c, hd(dw.embedding), layers, hd(dw.final_norm), np.zeros((c.d_model, 1)))


def boundary_margin(oracle_scores, got_scores, k):
    """(gap between the k-th and (k+1)-th oracle scores) / (max |score error|)."""
    s = np.sort(oracle_scores)[::-1]
    gap = s[k - 1] - s[k]
    err = np.max(np.abs(got_scores - oracle_scores))
    return gap / max(err, 1e-300), gap / s[k - 1], err / s[k - 1]


def _shape_case(name, layers):
    import paper_2603_05353_b200 as P

    if name == "llama3_8b":
        cfg = dataclasses.replace(P.llama3_8b_config(), n_layers=layers)
        task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=2048, prompt_length=32,
                               vocab_size=cfg.vocab_size)
    else:
        cfg = dataclasses.replace(P.qwen25vl_7b_config(), n_layers=layers)
        lens = [1280] * 24 + [512] * 4
        task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=None,
                               boundaries=tuple(np.cumsum(lens)[:-1].tolist()), prompt_length=32,
                               vocab_size=cfg.vocab_size)
    dw = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
    g = P.generate_task(task, seed=0)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    return P, cfg, dw, g, kvs


@pytest.mark.parametrize("shape", ["llama3_8b", "qwen25vl_7b"])
def test_headline_width_selection_matches_oracle(cuda, shape):
    P, cfg, dw, g, kvs = _shape_case(shape, layers=4)
    nl = P.default_norm_layer(cfg.n_layers)  # 2
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
    got_scores, got = res.scores_numpy().astype(np.float64), res.selected_numpy()
    ow = oracle_weights(dw, nl + 1)
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
    k = math.ceil(0.15 * 32768)
    margin, gap_rel, err_rel = boundary_margin(scores, got_scores, k)
    print(f"{shape}: k={k} boundary gap {gap_rel:.2e} rel, max score error {err_rel:.2e} rel, margin {margin:.1f}x; "
          f"max elementwise rel err {np.max(np.abs(got_scores - scores) / scores):.2e}")
    assert np.all(scores > 0)
    np.testing.assert_allclose(got_scores, scores, rtol=1e-4, atol=0)
    np.testing.assert_array_equal(sel, np.sort(O.select_topk(scores, k)))
    assert_same_selection(got, got_scores, scores, k, tag=shape)


def test_c3_reorder_64_chunks_matches_oracle(cuda):
    import paper_2603_05353_b200 as P

    cfg = dataclasses.replace(P.llama3_8b_config(), n_layers=2)
    task = P.SyntheticTask(kind="uniform_noise", total_length=131072, fixed_size=2048, prompt_length=32,
                           vocab_size=cfg.vocab_size)
    dw = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
    g = P.generate_task(task, seed=0)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    budget = math.ceil(0.15 * 131072)
    plan, _, second = P.reorder_and_reselect(dw, g.chunks, g.prompt_token_ids, budget=budget, prefilled=kvs)
    ow = oracle_weights(dw, 2)
    ochunks = [oracle_chunk(c) for c in kvs]
    perm, imps, _, scores, sel = O.reorder_and_reselect(ow, ochunks, g.prompt_token_ids, budget)
    srt = np.sort(imps)
    print(f"C3: 64 chunks, min relative importance gap {np.min(np.diff(srt) / srt[1:]):.2e}, "
          f"max importance rel err {np.max(np.abs(plan.chunk_importance - imps) / imps):.2e}")
    np.testing.assert_allclose(plan.chunk_importance, imps, rtol=1e-4)
    if assert_same_permutation(plan.permutation, perm, imps, plan.chunk_importance, tag="C3"):
        # near-tied chunks traded places: the second pass is checked against the
        # oracle's second pass over the same (our) order (reorder.py:150-181)
        cache = O.assemble([ochunks[i] for i in plan.permutation])
        ctx, prm = O.assign_positions("GLOBAL", cache.chunk_lengths, len(g.prompt_token_ids), None,
                                      cfg.max_position)
        scores = O.score_attention_norm(ow, cache, g.prompt_token_ids, np.concatenate(ctx), prm,
                                        P.default_norm_layer(cfg.n_layers))
    np.testing.assert_allclose(second.scores_numpy(), scores, rtol=1e-4, atol=0)
    assert_same_selection(second.selected_numpy(), second.scores_numpy(), scores, budget, tag="C3 second pass")


def test_depth_32_layers_c1_width_matches_oracle(cuda):
    import paper_2603_05353_b200 as P

    cfg = dataclasses.replace(P.c1_config(), n_layers=32)
    dw = P.DeviceWeights.from_host(P.init_weights(cfg, 7), "bf16")
    ow = dw.to_host()
    task = P.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32, vocab_size=1024)
    g = P.generate_task(task, 0)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)  # norm layer 19
    np.testing.assert_allclose(res.scores_numpy(), scores, rtol=1e-4, atol=0)
    np.testing.assert_array_equal(res.selected_numpy(), sel)
    want = O.recompute_selected(ow, oc, *O.make_plan(oc.context_length, sel))
    wk, wv = O.decode_view(want, cfg.rope_base)
    out = P.recompute_selected(dw, cache, P.make_plan(cache, res.selected))
    gk, gv = (to_np(t) for t in P.decode_view(out, cfg.rope_base))
    def frob(a, b):
        return float(np.linalg.norm(a - b) / np.linalg.norm(b))

    errs = [(rel_err(gk[li][sel], wk[li][sel]), rel_err(gv[li][sel], wv[li][sel])) for li in range(cfg.n_layers)]
    frobs = [(frob(gk[li][sel], wk[li][sel]), frob(gv[li][sel], wv[li][sel])) for li in range(cfg.n_layers)]
    print("recomputed-row K/V max-norm error by layer: " + " ".join(f"{li}:{max(e):.1e}" for li, e in enumerate(errs)))
    print("recomputed-row K/V Frobenius error by layer: " + " ".join(f"{li}:{max(e):.1e}" for li, e in enumerate(frobs)))
    assert max(max(e) for e in frobs) <= 1e-2
    assert max(max(e) for e in errs) <= 1.5e-2


@pytest.mark.parametrize("shape", ["llama3_8b"])
def test_headline_width_fp64_selection_bit_exact(cuda, shape):
    """score_precision='fp64' (exact.py): the scoring pass in float64 on the
    GPU reproduces the float64 reference's scores to ~1e-12 and its selected
    set bit for bit, whatever the boundary margin (selection.py:127-183)."""
    P, cfg, dw, g, kvs = _shape_case(shape, layers=4)
    nl = P.default_norm_layer(cfg.n_layers)
    cache = P.assemble(kvs)
    res = P.run_selection(dw, g.chunks, cache, g.prompt_token_ids,
                          P.SelectionConfig(ratio=0.15, score_precision="fp64"))
    got_scores, got = res.scores_numpy(), res.selected_numpy()
    ow = oracle_weights(dw, nl + 1)
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
    k = math.ceil(0.15 * 32768)
    s = np.sort(scores)[::-1]
    print(f"{shape} fp64: boundary gap {(s[k - 1] - s[k]) / s[k - 1]:.2e} rel, max score rel err "
          f"{np.max(np.abs(got_scores - scores) / scores):.2e}")
    np.testing.assert_allclose(got_scores, scores, rtol=1e-10, atol=0)
    np.testing.assert_array_equal(got, sel)


def test_c3_reorder_64_chunks_fp64_bit_exact(cuda):
    """reorder_and_reselect(score_precision='fp64') at 64 x 2048 chunks
    (128K): importances to ~1e-12 of the float64 oracle, the permutation and
    the second-pass set bit-exact at any margin (reorder.py:116-181)."""
    import paper_2603_05353_b200 as P

    cfg = dataclasses.replace(P.llama3_8b_config(), n_layers=2)
    task = P.SyntheticTask(kind="uniform_noise", total_length=131072, fixed_size=2048, prompt_length=32,
                           vocab_size=cfg.vocab_size)
    dw = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
    g = P.generate_task(task, seed=0)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    budget = math.ceil(0.15 * 131072)
    plan, _, second = P.reorder_and_reselect(dw, g.chunks, g.prompt_token_ids, budget=budget, prefilled=kvs,
                                             score_precision="fp64")
    ow = oracle_weights(dw, 2)
    perm, imps, _, scores, sel = O.reorder_and_reselect(ow, [oracle_chunk(c) for c in kvs], g.prompt_token_ids,
                                                        budget)
    np.testing.assert_allclose(plan.chunk_importance, imps, rtol=1e-10)
    np.testing.assert_array_equal(plan.permutation, perm)
    np.testing.assert_allclose(second.scores_numpy(), scores, rtol=1e-10, atol=0)
    np.testing.assert_array_equal(second.selected_numpy(), sel)
