"""paper_2603_05353_b200: B200-native InfoFlow-KV query-time context assembly.

Drop-in for the reference package ``chunkkv`` (0.1.0) on its hot path:
precompute per-chunk KV under chunk-local RoPE, then ``assemble`` ->
``run_selection`` (attention-norm scoring + exact top-k) ->
``make_plan`` / ``recompute_selected``, optionally ``reorder_and_reselect``.
The names, argument meanings and exceptions are the reference's
(chunkkv/__init__.py:3-81); tensors live in HBM and every compute step is an
sm_100a kernel behind the C ABI in ``include/ifkv.h`` (no CPU fallback).
"""

from .cache import (
    AssembledCache,
    ChunkKV,
    FidelityReport,
    PromptKV,
    Provenance,
    assemble,
    cache_fidelity,
    decode_view,
    full_prefill,
    prefill_chunk,
    prefill_chunks,
    replace_entries,
    to_decode_layout,
)
from .decode import first_token_logits, greedy_token
from .errors import ChunkKVError, ConfigurationError, DataFormatError, NativeError
from .model import (
    DeviceWeights,
    ModelConfig,
    Weights,
    c1_config,
    init_weights,
    llama3_8b_config,
    qwen25vl_7b_config,
    toy_config,
)
from .pipeline import PathResult, QueryGraph, StageTimer, assemble_select_recompute, query_graph
from .positions import ChunkSpec, GeometryConfig, GeometryMode, PositionAssignment, assign_positions
from .recompute import RecomputePlan, make_plan, recompute_selected
from .reorder import ReorderPlan, reorder_and_reselect, score_chunks
from .selection import (
    SelectionConfig,
    SelectionResult,
    Strategy,
    default_norm_layer,
    run_selection,
    score_attention_norm,
    score_cacheblend,
    score_from_attention,
    select_epic,
    select_random,
    select_topk,
)
from .storage import load_cache, save_cache
from .tasks import GeneratedTask, SyntheticTask, generate_task, make_chunks

__version__ = "0.1.0"
