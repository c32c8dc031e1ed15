"""Pin the oracle and the host-side restatements against golden vectors
produced by the reference itself (tests/golden/make_golden.py).

Integer results (selected sets, permutations, token ids) must be identical;
float64 results agree to 1e-9 (summation order differs: blocked attention,
GQA grouping)."""

import hashlib

import numpy as np
import pytest

import oracle as O
from paper_2603_05353_b200.model import ModelConfig, bf16_round, init_weights
from paper_2603_05353_b200.positions import ChunkSpec, GeometryConfig, assign_positions
from paper_2603_05353_b200.tasks import SyntheticTask, generate_task

TINY = ModelConfig(n_layers=2, n_heads=2, d_model=16, d_head=8, d_ff=32, vocab_size=64, max_position=4096)
C1 = ModelConfig(n_layers=2, n_heads=4, d_model=512, d_head=128, d_ff=1792, vocab_size=1024, max_position=8192)
GQA = ModelConfig(n_layers=2, n_heads=4, d_model=64, d_head=16, d_ff=96, vocab_size=128, max_position=4096,
                  n_kv_heads=2)


def tensor_hash(weights) -> str:
    h = hashlib.sha256()
    for name, t in weights.named_tensors():
        h.update(name.encode())
        h.update(np.ascontiguousarray(t, dtype=np.float64).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def tiny_w():
    return init_weights(TINY, seed=7)


def _oracle_chunks(w, toks, lens):
    out, s = [], 0
    for i, n in enumerate(lens):
        out.append(O.prefill_chunk(w, f"c{i}", toks[s:s + n]))
        s += n
    return out


class TestHostRestatements:
    def test_init_weights_bit_identical(self, golden_small, tiny_w):
        assert tensor_hash(tiny_w) == str(golden_small["tiny_weights_hash"])
        assert tensor_hash(init_weights(C1, seed=7)) == str(golden_small["c1_weights_hash_f64"])

    def test_gqa_init_matches_generator(self, golden_small):
        assert tensor_hash(init_weights(GQA, seed=11)) == str(golden_small["gqa_weights_hash"])

    def test_bf16_rounded_c1_weights(self, golden_c1):
        w = init_weights(C1, seed=7).bf16_rounded()
        assert tensor_hash(w) == str(golden_c1["c1_weights_hash_bf16"])

    def test_generate_task(self, golden_small):
        specs = [("uniform_noise", 2048, 256, 32), ("needle", 256, 64, 8), ("needle", 128, 32, 8)]
        for i, (kind, n, fs, pl) in enumerate(specs):
            t = SyntheticTask(kind=kind, total_length=n, fixed_size=fs, prompt_length=pl,
                              vocab_size=1024 if kind == "uniform_noise" else 256)
            for seed in (0, 5):
                g = generate_task(t, seed)
                np.testing.assert_array_equal(np.concatenate([c.token_ids for c in g.chunks]),
                                              golden_small[f"task{i}_s{seed}_tokens"])
                np.testing.assert_array_equal(g.prompt_token_ids, golden_small[f"task{i}_s{seed}_prompt"])
                want = int(golden_small[f"task{i}_s{seed}_needle"])
                assert (g.needle_index if g.needle_index is not None else -1) == want

    @pytest.mark.parametrize("mode,off", [("GLOBAL", None), ("HL-HP", None), ("HL-TP", 200), ("TL-TP", 200)])
    def test_assign_positions(self, golden_small, mode, off):
        toks = golden_small["tiny_tokens"]
        chunks = [ChunkSpec(f"c{i}", toks[8 * i:8 * i + 8], i) for i in range(3)]
        a = assign_positions(GeometryConfig(mode=mode, prompt_length=4, chunk_lengths=(8, 8, 8), prompt_offset=off),
                             chunks)
        got = np.concatenate([a.context_concat(), a.prompt_positions])
        np.testing.assert_array_equal(got, golden_small[f"tiny_pos_{mode}"])
        ctx, prm = O.assign_positions(mode, (8, 8, 8), 4, off)
        np.testing.assert_array_equal(np.concatenate(ctx + [prm]), golden_small[f"tiny_pos_{mode}"])

    def test_topk_brute_force_vectors(self, golden_small):
        for vec, (n, k), sel in zip(golden_small["topk_vecs"], golden_small["topk_nk"], golden_small["topk_sel"]):
            got = O.select_topk(vec[:n], int(k))
            np.testing.assert_array_equal(got, sel[:k])


@pytest.fixture(scope="module")
def setup(golden_small, tiny_w):
    toks = golden_small["tiny_tokens"]
    chunks = _oracle_chunks(tiny_w, toks, [8, 8, 8])
    return toks, golden_small["tiny_prompt"], chunks, O.assemble(chunks)


class TestOracleTiny:

    def test_prefill_chunks(self, golden_small, setup):
        _, _, chunks, _ = setup
        np.testing.assert_allclose(np.stack([c.keys for c in chunks]), golden_small["tiny_chunk_keys"], atol=1e-12)
        np.testing.assert_allclose(np.stack([c.values for c in chunks]), golden_small["tiny_chunk_values"],
                                   atol=1e-12)

    @pytest.mark.parametrize("mode,off", [("GLOBAL", None), ("HL-HP", None), ("HL-TP", 200), ("TL-TP", 200)])
    def test_scores_and_topk(self, golden_small, tiny_w, setup, mode, off):
        _, prompt, _, cache = setup
        ctx, prm = O.assign_positions(mode, (8, 8, 8), 4, off)
        s = O.score_attention_norm(tiny_w, cache, prompt, np.concatenate(ctx), prm, 1)
        np.testing.assert_allclose(s, golden_small[f"tiny_scores_{mode}"], rtol=1e-9, atol=1e-12)
        np.testing.assert_array_equal(O.select_topk(s, 6), golden_small[f"tiny_sel6_{mode}"])

    def test_recompute(self, golden_small, tiny_w, setup):
        _, _, _, cache = setup
        sel, pos, upto = O.make_plan(cache.context_length, [3, 11, 20])
        rec = O.recompute_selected(tiny_w, cache, sel, pos, upto)
        np.testing.assert_allclose(rec.keys, golden_small["tiny_rec_keys"], atol=1e-10)
        np.testing.assert_allclose(rec.values, golden_small["tiny_rec_values"], atol=1e-10)
        dk, _ = O.decode_view(rec, TINY.rope_base)
        np.testing.assert_allclose(dk, golden_small["tiny_rec_decode_keys"], atol=1e-10)

    def test_full_prefill_and_fidelity(self, golden_small, tiny_w, setup):
        toks, _, _, cache = setup
        full = O.full_prefill(tiny_w, toks)
        np.testing.assert_allclose(full.keys, golden_small["tiny_full_keys"], atol=1e-10)
        fro, _ = O.fidelity(cache, full, TINY.rope_base)
        assert fro == pytest.approx(float(golden_small["tiny_fidelity_before"][0]), rel=1e-9)
        sel, pos, upto = O.make_plan(cache.context_length, np.arange(24))
        rec = O.recompute_selected(tiny_w, cache, sel, pos, upto)
        _, worst = O.fidelity(rec, full, TINY.rope_base)
        assert worst <= 1e-10 + float(golden_small["tiny_full_recompute_maxabs"][0])

    @pytest.mark.parametrize("budget", [1, 6, 12])
    def test_reorder(self, golden_small, tiny_w, setup, budget):
        _, prompt, chunks, _ = setup
        perm, imps, _, scores, sel = O.reorder_and_reselect(tiny_w, chunks, prompt, budget)
        np.testing.assert_array_equal(perm, golden_small[f"tiny_reorder{budget}_perm"])
        np.testing.assert_allclose(imps, golden_small[f"tiny_reorder{budget}_imp"], rtol=1e-9)
        np.testing.assert_array_equal(sel, golden_small[f"tiny_reorder{budget}_sel"])
        np.testing.assert_allclose(scores, golden_small[f"tiny_reorder{budget}_scores"], rtol=1e-9, atol=1e-12)

    @pytest.mark.parametrize("mode", ["mean", "max"])
    def test_chunk_score_modes(self, golden_small, tiny_w, setup, mode):
        _, prompt, chunks, _ = setup
        imps, _ = O.chunk_importance(tiny_w, chunks, prompt, 6, chunk_score=mode)
        np.testing.assert_allclose(imps, golden_small[f"tiny_imp_{mode}"], rtol=1e-9)


class TestOracleGQA:
    def test_gqa_matches_tiled_mha_reference(self, golden_small):
        w = init_weights(GQA, seed=11)
        toks, prompt = golden_small["gqa_tokens"], golden_small["gqa_prompt"]
        chunks = _oracle_chunks(w, toks, [32, 32, 32])
        np.testing.assert_allclose(np.stack([c.keys for c in chunks]), golden_small["gqa_chunk_keys"], atol=1e-11)
        cache = O.assemble(chunks)
        scores, sel = O.run_selection(w, cache, prompt, ratio=0.2)
        np.testing.assert_allclose(scores, golden_small["gqa_scores"], rtol=1e-9, atol=1e-12)
        np.testing.assert_array_equal(sel, golden_small["gqa_selected"])
        s, p, u = O.make_plan(cache.context_length, sel)
        rec = O.recompute_selected(w, cache, s, p, u)
        np.testing.assert_allclose(rec.keys, golden_small["gqa_rec_keys"], atol=1e-10)
        np.testing.assert_allclose(rec.values, golden_small["gqa_rec_values"], atol=1e-10)


@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_c1_bf16_weights(golden_c1, seed):
    """BASELINE config 1 (Dh = 128, 8 x 256 + 32, r = 0.15) on bf16-valued weights."""
    p = f"c1s{seed}_"
    w = init_weights(C1, seed=7).bf16_rounded()
    toks = golden_c1[p + "tokens"]
    chunks = _oracle_chunks(w, toks, [256] * 8)
    stats = np.stack([np.array([[k.sum(), np.abs(k).sum(), (k * k).sum()] for k in c.keys]) for c in chunks]
                     + [np.array([[v.sum(), np.abs(v).sum(), (v * v).sum()] for v in c.values]) for c in chunks])
    np.testing.assert_allclose(stats, golden_c1[p + "chunk_kv_stats"], rtol=1e-9, atol=1e-9)
    cache = O.assemble(chunks)
    scores, sel = O.run_selection(w, cache, golden_c1[p + "prompt"], ratio=0.15)
    np.testing.assert_allclose(scores, golden_c1[p + "scores"], rtol=1e-9, atol=1e-13)
    np.testing.assert_array_equal(sel, golden_c1[p + "selected"])
    s, pp, u = O.make_plan(cache.context_length, sel)
    rec = O.recompute_selected(w, cache, s, pp, u)
    dk, dv = O.decode_view(rec, C1.rope_base)
    rows = golden_c1[p + "sample_rows"]
    np.testing.assert_allclose(dk[:, rows], golden_c1[p + "rec_key_rows"], atol=1e-9)
    np.testing.assert_allclose(dv[:, rows], golden_c1[p + "rec_value_rows"], atol=1e-9)
    perm, imps, _, _, sel2 = O.reorder_and_reselect(w, chunks, golden_c1[p + "prompt"], 308)
    np.testing.assert_array_equal(perm, golden_c1[p + "reorder_perm"])
    np.testing.assert_allclose(imps, golden_c1[p + "reorder_imp"], rtol=1e-9)
    np.testing.assert_array_equal(sel2, golden_c1[p + "reorder_sel"])


class TestOracleCacheBlend:
    """Baseline selector (selection.py:190-223) pinned to the reference's scores."""

    @pytest.mark.parametrize("early", [1, 2])
    def test_tiny_scores(self, golden_small, tiny_w, early):
        toks = golden_small["tiny_tokens"]
        s = O.score_cacheblend(tiny_w, [toks[8 * i:8 * i + 8] for i in range(3)], early)
        np.testing.assert_allclose(s, golden_small[f"tiny_cacheblend{early}_scores"], rtol=1e-9, atol=1e-12)
        if early == 2:
            np.testing.assert_array_equal(O.select_topk(s, 6), golden_small["tiny_cacheblend_sel6"])

    def test_c1_scores_and_selection(self, golden_c1):
        w = init_weights(C1, seed=7).bf16_rounded()
        toks = golden_c1["c1s0_tokens"]
        s = O.score_cacheblend(w, [toks[256 * i:256 * i + 256] for i in range(8)], 2)
        np.testing.assert_allclose(s, golden_c1["c1s0_cacheblend_scores"], rtol=1e-9, atol=1e-12)
        np.testing.assert_array_equal(O.select_topk(s, 308), golden_c1["c1s0_cacheblend_selected"])

    def test_single_chunk_scores_zero(self, tiny_w):
        s = O.score_cacheblend(tiny_w, [np.arange(10) % 64], 2)
        np.testing.assert_array_equal(s, np.zeros(10))
