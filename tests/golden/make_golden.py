"""Generate golden vectors by running the REFERENCE (chunkkv 0.1.0) itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  tests/test_oracle_golden.py pins the oracle
(oracle/ifkv_oracle.py) and the host-side restatements (init_weights,
generate_task, assign_positions) against these files.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))

import chunkkv as ck  # noqa: E402
from chunkkv import cache as ck_cache  # noqa: E402

from paper_2603_05353_b200.model import bf16_round  # noqa: E402
from paper_2603_05353_b200.model import init_weights as prod_init  # noqa: E402
from paper_2603_05353_b200.model import ModelConfig as ProdConfig  # noqa: E402


def tensor_hash(weights) -> str:
    h = hashlib.sha256()
    for name, t in weights.named_tensors():
        h.update(name.encode())
        h.update(np.ascontiguousarray(t, dtype=np.float64).tobytes())
    return h.hexdigest()


def ref_weights_from(arrs_cfg, layers, embedding, final_norm, out_head):
    return ck.Weights(config=arrs_cfg, embedding=embedding, layers=layers, final_norm=final_norm, out_head=out_head)


def rounded(w):
    layers = [ck.model.LayerWeights(**{n: bf16_round(t) for n, t in lw.tensors()}) for lw in w.layers]
    return ck.Weights(config=w.config, embedding=bf16_round(w.embedding), layers=layers,
                      final_norm=bf16_round(w.final_norm), out_head=bf16_round(w.out_head))


def kv_stats(keys_list):
    """Per-layer (sum, sum|x|, sum x^2) of a list of (T, H, Dh) arrays."""
    return np.array([[k.sum(), np.abs(k).sum(), (k * k).sum()] for k in keys_list])


def tiny_case(out):
    cfg = ck.ModelConfig(n_layers=2, n_heads=2, d_model=16, d_head=8, d_ff=32, vocab_size=64, max_position=4096)
    w = ck.init_weights(cfg, seed=7)
    out["tiny_weights_hash"] = np.array(tensor_hash(w))
    rng = np.random.default_rng(8)
    toks = rng.integers(0, 64, 24)
    prompt = rng.integers(0, 64, 4)
    chunks = [ck.ChunkSpec(f"c{i}", toks[8 * i:8 * i + 8], i) for i in range(3)]
    kvs = [ck.prefill_chunk(w, c) for c in chunks]
    cache = ck.assemble(kvs)
    out["tiny_tokens"], out["tiny_prompt"] = toks, prompt
    out["tiny_chunk_keys"] = np.stack([np.stack(c.keys) for c in kvs])  # (K, L, len, H, Dh)
    out["tiny_chunk_values"] = np.stack([np.stack(c.values) for c in kvs])
    for mode, off in (("GLOBAL", None), ("HL-HP", None), ("HL-TP", 200), ("TL-TP", 200)):
        g = ck.GeometryConfig(mode=mode, prompt_length=4, chunk_lengths=(8, 8, 8), prompt_offset=off)
        a = ck.assign_positions(g, chunks)
        out[f"tiny_pos_{mode}"] = np.concatenate([a.context_concat(), a.prompt_positions])
        s = ck.score_attention_norm(w, cache, prompt, a, norm_layer=1)
        out[f"tiny_scores_{mode}"] = s
        out[f"tiny_sel6_{mode}"] = ck.select_topk(s, 6)
    plan = ck.make_plan(cache, np.array([3, 11, 20]))
    rec = ck.recompute_selected(w, cache, plan)
    out["tiny_rec_keys"] = np.stack(rec.keys)
    out["tiny_rec_values"] = np.stack(rec.values)
    dk, dv = ck.decode_view(rec, cfg.rope_base)
    out["tiny_rec_decode_keys"] = np.stack(dk)
    full = ck.full_prefill(w, toks)
    out["tiny_full_keys"] = np.stack(full.keys)
    out["tiny_fidelity_before"] = np.array([ck.cache_fidelity(cache, full, cfg.rope_base).frobenius])
    out["tiny_fidelity_after"] = np.array([ck.cache_fidelity(rec, full, cfg.rope_base).frobenius])
    all_plan = ck.make_plan(cache, np.arange(24))
    rec_all = ck.recompute_selected(w, cache, all_plan)
    out["tiny_full_recompute_maxabs"] = np.array([ck.cache_fidelity(rec_all, full, cfg.rope_base).max_abs])
    for budget in (1, 6, 12):
        plan_r, cache_r, second = ck.reorder_and_reselect(w, chunks, prompt, budget=budget, prefilled=kvs)
        out[f"tiny_reorder{budget}_perm"] = plan_r.permutation
        out[f"tiny_reorder{budget}_imp"] = plan_r.chunk_importance
        out[f"tiny_reorder{budget}_sel"] = second.selected
        out[f"tiny_reorder{budget}_scores"] = second.scores
    for mode in ("mean", "max"):
        imps, _ = ck.score_chunks(w, chunks, prompt, budget=6, chunk_score=mode, prefilled=kvs)
        out[f"tiny_imp_{mode}"] = imps
    # baseline selector: CacheBlend early-layer deviation (selection.py:190-223)
    for el in (1, 2):
        out[f"tiny_cacheblend{el}_scores"] = ck.selection.score_cacheblend(w, chunks, el)
    cb = ck.run_selection(w, chunks, cache, prompt, ck.SelectionConfig(strategy="cacheblend", topk=6,
                                                                        cacheblend_layers=2))
    out["tiny_cacheblend_sel6"] = cb.selected
    # IFKC files written by the reference (f64 and f32 precision codes)
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        ck.save_cache(kvs[1], Path(d) / "a.ifkc")
        out["tiny_ifkc_f64"] = np.frombuffer((Path(d) / "a.ifkc").read_bytes(), dtype=np.uint8)
        w32 = ck.init_weights(cfg, seed=3, precision="f32")
        c32 = ck.prefill_chunk(w32, ck.ChunkSpec("f32chunk", np.arange(5)))
        ck.save_cache(c32, Path(d) / "b.ifkc")
        out["tiny_ifkc_f32"] = np.frombuffer((Path(d) / "b.ifkc").read_bytes(), dtype=np.uint8)
        out["tiny_ifkc_f32_keys"] = np.stack(c32.keys)


def c1_case(out, seed):
    cfg = ck.ModelConfig(n_layers=2, n_heads=4, d_model=512, d_head=128, d_ff=1792, vocab_size=1024,
                         rope_base=10000.0, max_position=8192)
    w = rounded(ck.init_weights(cfg, seed=7))
    if seed == 0:
        out["c1_weights_hash_bf16"] = np.array(tensor_hash(w))
    task = ck.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32,
                            vocab_size=1024)
    g = ck.generate_task(task, seed)
    kvs = [ck.prefill_chunk(w, c) for c in g.chunks]
    cache = ck.assemble(kvs)
    p = f"c1s{seed}_"
    out[p + "tokens"] = np.concatenate([c.token_ids for c in g.chunks])
    out[p + "prompt"] = g.prompt_token_ids
    out[p + "chunk_kv_stats"] = np.stack([kv_stats(c.keys) for c in kvs] + [kv_stats(c.values) for c in kvs])
    sel = ck.run_selection(w, g.chunks, cache, g.prompt_token_ids, ck.SelectionConfig(ratio=0.15))
    out[p + "scores"] = sel.scores
    out[p + "selected"] = sel.selected
    rec = ck.recompute_selected(w, cache, ck.make_plan(cache, sel.selected))
    dk, dv = ck.decode_view(rec, cfg.rope_base)
    out[p + "rec_key_stats"] = kv_stats(dk)
    out[p + "rec_value_stats"] = kv_stats(dv)
    rows = np.array([0, 1, 255, 256, 1000, 2047])
    rows = np.union1d(rows, sel.selected[::37])
    out[p + "sample_rows"] = rows
    out[p + "rec_key_rows"] = np.stack([k[rows] for k in dk])
    out[p + "rec_value_rows"] = np.stack([v[rows] for v in dv])
    plan_r, cache_r, second = ck.reorder_and_reselect(w, g.chunks, g.prompt_token_ids, budget=308, prefilled=kvs)
    out[p + "reorder_perm"] = plan_r.permutation
    out[p + "reorder_imp"] = plan_r.chunk_importance
    out[p + "reorder_sel"] = second.selected
    if seed == 0:
        cb = ck.run_selection(w, g.chunks, cache, g.prompt_token_ids,
                              ck.SelectionConfig(strategy="cacheblend", ratio=0.15, cacheblend_layers=2))
        out[p + "cacheblend_scores"] = cb.scores
        out[p + "cacheblend_selected"] = cb.selected


def gqa_case(out):
    """GQA (H=4, Hkv=2) via the reference's MHA with tiled wk/wv (SURVEY §7 hard part 5)."""
    pcfg = ProdConfig(n_layers=2, n_heads=4, d_model=64, d_head=16, d_ff=96, vocab_size=128, rope_base=10000.0,
                      max_position=4096, n_kv_heads=2)
    pw = prod_init(pcfg, seed=11)
    out["gqa_weights_hash"] = np.array(tensor_hash(pw))
    rcfg = ck.ModelConfig(n_layers=2, n_heads=4, d_model=64, d_head=16, d_ff=96, vocab_size=128, rope_base=10000.0,
                          max_position=4096)
    grp, dh = 2, 16

    def tile(wkv):  # (d, Hkv*Dh) -> (d, H*Dh): head h reads kv head h // grp
        blocks = [wkv[:, (h // grp) * dh:(h // grp + 1) * dh] for h in range(4)]
        return np.concatenate(blocks, axis=1)

    layers = [ck.model.LayerWeights(attn_norm=lw.attn_norm, wq=lw.wq, wk=tile(lw.wk), wv=tile(lw.wv), wo=lw.wo,
                                    mlp_norm=lw.mlp_norm, w_gate=lw.w_gate, w_up=lw.w_up, w_down=lw.w_down)
              for lw in pw.layers]
    w = ck.Weights(config=rcfg, embedding=pw.embedding, layers=layers, final_norm=pw.final_norm,
                   out_head=pw.out_head)
    rng = np.random.default_rng(3)
    toks = rng.integers(0, 128, 96)
    prompt = rng.integers(0, 128, 8)
    chunks = [ck.ChunkSpec(f"c{i}", toks[32 * i:32 * i + 32], i) for i in range(3)]
    kvs = [ck.prefill_chunk(w, c) for c in chunks]
    cache = ck.assemble(kvs)
    out["gqa_tokens"], out["gqa_prompt"] = toks, prompt
    # MHA keys of head h equal GQA kv head h // grp: keep kv heads 0 and 2
    out["gqa_chunk_keys"] = np.stack([np.stack(c.keys)[:, :, ::grp] for c in kvs])
    sel = ck.run_selection(w, chunks, cache, prompt, ck.SelectionConfig(ratio=0.2))
    out["gqa_scores"], out["gqa_selected"] = sel.scores, sel.selected
    rec = ck.recompute_selected(w, cache, ck.make_plan(cache, sel.selected))
    out["gqa_rec_keys"] = np.stack(rec.keys)[:, :, ::grp]
    out["gqa_rec_values"] = np.stack(rec.values)[:, :, ::grp]


def tasks_case(out):
    for i, (kind, n, fs, pl) in enumerate([("uniform_noise", 2048, 256, 32), ("needle", 256, 64, 8),
                                           ("needle", 128, 32, 8)]):
        t = ck.SyntheticTask(kind=kind, total_length=n, fixed_size=fs, prompt_length=pl,
                             vocab_size=1024 if kind == "uniform_noise" else 256)
        for seed in (0, 5):
            g = ck.generate_task(t, seed)
            out[f"task{i}_s{seed}_tokens"] = np.concatenate([c.token_ids for c in g.chunks])
            out[f"task{i}_s{seed}_prompt"] = g.prompt_token_ids
            out[f"task{i}_s{seed}_needle"] = np.array(-1 if g.needle_index is None else g.needle_index)
    c1 = ck.init_weights(ck.ModelConfig(n_layers=2, n_heads=4, d_model=512, d_head=128, d_ff=1792,
                                        vocab_size=1024, rope_base=10000.0, max_position=8192), seed=7)
    out["c1_weights_hash_f64"] = np.array(tensor_hash(c1))
    # top-k brute-force vectors with heavy ties (selection.py:172-183)
    rng = np.random.default_rng(0)
    vecs, ks, sels = [], [], []
    for _ in range(200):
        n = int(rng.integers(1, 40))
        s = rng.choice([0.1, 0.25, 0.5, 0.77], size=n)
        k = int(rng.integers(0, n + 1))
        vecs.append(np.pad(s, (0, 40 - n), constant_values=np.nan))
        ks.append((n, k))
        sels.append(np.pad(ck.select_topk(s, k), (0, 40 - k), constant_values=-1))
    out["topk_vecs"], out["topk_nk"], out["topk_sel"] = np.stack(vecs), np.array(ks), np.stack(sels)


def main():
    out = {}
    tasks_case(out)
    tiny_case(out)
    gqa_case(out)
    np.savez_compressed(HERE / "golden_small.npz", **out)
    out = {}
    for seed in (0, 1):
        c1_case(out, seed)
    np.savez_compressed(HERE / "golden_c1.npz", **out)
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
