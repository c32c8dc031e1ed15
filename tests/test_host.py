"""CPU-side checks: the C-ABI library loads and exports every entry point of
include/ifkv.h; host logic (configs, positions, plans, work-item planning)
behaves like the reference; the product fails loudly without a GPU."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2603_05353_b200 as P
from paper_2603_05353_b200 import _native as N
from paper_2603_05353_b200 import engine as E

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "ifkv.h").read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(ifkv_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    from paper_2603_05353_b200.build import LIB, build

    build()
    lib = N.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.ifkv_abi_version() == 1
    assert set(syms) <= set(N.EXPORTS)


def test_argument_errors_map_to_configuration_error():
    # rope_table validates before touching the device: d_head must be even
    with pytest.raises(P.ConfigurationError):
        N.call("ifkv_rope_table", None, 4, 7, 10000.0, None, None)
    # the newer entry points validate their shapes before any CUDA call too
    with pytest.raises(P.ConfigurationError):  # rows must be a multiple of 32
        N.call("ifkv_prompt_mm", None, 3, 16, 4096, None, 4096, 1, None, None)
    with pytest.raises(P.ConfigurationError):  # splits > K / 64
        N.call("ifkv_prompt_mm", None, 3, 32, 128, None, 4096, 3, None, None)
    with pytest.raises(P.ConfigurationError):
        N.call("ifkv_merge_partials", None, None, 0, 10, 128, None, None, None)
    with pytest.raises(P.ConfigurationError):
        N.call("ifkv_merge_prompt_states", None, None, 2, 1, 32, 8, 126, None, None, None)


def test_model_config_validation():
    with pytest.raises(P.ConfigurationError):
        P.ModelConfig(n_layers=1, n_heads=3, d_model=12, d_head=4, d_ff=8, vocab_size=10, n_kv_heads=2)
    with pytest.raises(P.ConfigurationError):
        P.ModelConfig(n_layers=1, n_heads=2, d_model=10, d_head=4, d_ff=8, vocab_size=10)
    c = P.llama3_8b_config()
    assert c.kv_heads == 8 and c.params_per_layer() == 218_103_808


def test_selection_config_rules():
    with pytest.raises(P.ConfigurationError):
        P.SelectionConfig(topk=3, ratio=0.5)
    with pytest.raises(P.ConfigurationError):
        P.SelectionConfig()
    assert P.SelectionConfig(ratio=0.15).resolve_budget(32768) == 4916
    assert P.SelectionConfig(ratio=0.15).resolve_budget(2048) == 308
    assert P.default_norm_layer(32) == 19 and P.default_norm_layer(2) == 1 and P.default_norm_layer(1) == 0
    assert P.Strategy.parse("attention_norm") is P.Strategy.ATTENTION_NORM


def test_geometry_errors():
    chunks = P.make_chunks(np.arange(16), [8, 8])
    with pytest.raises(P.ConfigurationError):
        P.assign_positions(P.GeometryConfig(mode="tl-tp", prompt_length=2, chunk_lengths=(8, 8), prompt_offset=4),
                           chunks)
    with pytest.raises(P.ConfigurationError):
        P.assign_positions(P.GeometryConfig(mode="global", prompt_length=2, chunk_lengths=(8, 8), max_position=17),
                           chunks)
    with pytest.raises(P.ConfigurationError):
        P.GeometryMode.parse("sideways")


def test_plan_validation_host():
    with pytest.raises(P.ConfigurationError):
        P.RecomputePlan(selected=np.array([5, 2]), positions=np.array([5, 2]), allowed_upto=np.array([5, 2]))
    with pytest.raises(P.ConfigurationError):
        P.RecomputePlan(selected=np.array([5]), positions=np.array([5]), allowed_upto=np.array([4]))


def test_segments_and_work_items():
    d = np.array([0, 0, 5, 5, 5, 0, 9])
    assert E.segments_from_deltas(d, 10) == [(10, 2, 0), (12, 3, 5), (15, 1, 0), (16, 1, 9)]
    g = [E.PromptGroup(np.arange(4), np.arange(4), [(0, 300, 7), (300, 10, 0)]),
         E.PromptGroup(np.arange(4), np.arange(4), [(310, 5, 7)])]
    items, begin, n_ctx, qg, qc, deltas = E._plan_items(g, 4)
    assert deltas == [7]
    # context items first (group 0: 300 rows -> 128, 128, 44; then 10 rows; group 1: 5), then one prompt item per group
    assert begin.tolist() == [0, 4, 5] and n_ctx == 5
    assert items[:, 3].tolist() == [128, 128, 44, 10, 5, 4, 4]
    assert items[:, 4].tolist() == [0, 0, 0, 0, 0, 1, 1]
    assert items[:, 0].tolist() == [0, 0, 0, 0, 1, 0, 1]
    assert qg.tolist() == [0, 0, 1, 1] and qc.tolist() == [0, -1, 0, -1]
    # prompts longer than 128 tokens: the causal prompt keys split into <= 128-key items
    long = [E.PromptGroup(np.arange(300), np.arange(300), [(0, 10, 0)])]
    items, begin, n_ctx, _, _, _ = E._plan_items(long, 300)
    assert n_ctx == 1 and items[1:, 2].tolist() == [0, 128, 256] and items[1:, 3].tolist() == [128, 128, 44]
    assert items[1:, 4].tolist() == [1, 1, 1]


def test_score_from_attention_seam():
    a = np.array([[0.2, 0.5, 0.1], [0.3, 0.2, 0.4]])
    np.testing.assert_allclose(P.score_from_attention(a, 3), [0.5, 0.7, 0.5])
    h = np.stack([np.array([[1.0, 0.0, 0.0]]), np.array([[0.0, 1.0, 0.0]])])
    np.testing.assert_allclose(P.score_from_attention(h, 3), [0.5, 0.5, 0.0])


def test_epic_and_random_selectors():
    assert P.select_epic([4, 4], 0.25).tolist() == [0, 4]
    assert P.select_epic([10], 0.15).tolist() == [0, 1]
    np.testing.assert_array_equal(P.select_random(20, 5, 3), P.select_random(20, 5, 3))


def test_bf16_round_matches_torch():
    import torch

    x = np.random.default_rng(0).standard_normal(10000) * 10
    want = torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(P.model.bf16_round(x), want)


def test_device_ops_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        P.DeviceWeights.random(P.toy_config(), 0)


def test_score_precision_option():
    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200.errors import ConfigurationError

    assert P.SelectionConfig(ratio=0.1).score_precision == "fp32"
    assert P.SelectionConfig(ratio=0.1, score_precision="fp64").score_precision == "fp64"
    with pytest.raises(ConfigurationError):
        P.SelectionConfig(ratio=0.1, score_precision="fp16")
