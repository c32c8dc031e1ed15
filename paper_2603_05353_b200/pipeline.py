"""The timed path as one call: assemble -> (reorder) -> select -> recompute
(reference harness.py:433-456 minus chunk prefill and decode, which sit
outside the metric: prepared context, time to the recomputed cache).

``assemble_select_recompute`` is the public entry point the benchmark's
end-to-end leg calls; ``StageTimer`` records CUDA events between stages on
the current stream.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import engine as E
from .cache import AssembledCache, ChunkKV, assemble, assemble_decode_layout
from .positions import ChunkSpec
from .recompute import RecomputePlan, make_plan, recompute_selected
from .reorder import ReorderPlan, reorder_and_reselect
from .selection import (SelectionConfig, SelectionResult, Strategy, default_norm_layer, resolve_geometry,
                        run_selection, select_topk)
from .positions import assign_positions


class StageTimer:
    """CUDA-event marks on the current stream; durations read after a sync."""

    def __init__(self, enabled: bool = True):
        self.enabled = enabled
        self.marks: List = []

    def mark(self, name: str):
        if not self.enabled:
            return
        import torch

        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.marks.append((name, ev))

    def durations_ms(self) -> Dict[str, float]:
        out = {}
        for (_, a), (name, b) in zip(self.marks[:-1], self.marks[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


@dataclass
class PathResult:
    cache: AssembledCache
    selection: SelectionResult
    plan: RecomputePlan
    reorder: Optional[ReorderPlan] = None


# IFKV_STORE_OVERLAP=1: score on a high-priority stream while the gather runs
# (A/B: tools/path_ab.py measured no step-level difference, so off)
STORE_OVERLAP = os.environ.get("IFKV_STORE_OVERLAP", "0") == "1"


def _after_previous(stream):
    """An event marking everything enqueued on ``stream`` before the current
    query (the gather is enqueued after it, so waiting on it does not wait
    for the gather)."""
    import torch

    ev = torch.cuda.Event()
    ev.record(stream)
    return ev


def _shared_store(chunk_kvs: Sequence[ChunkKV]):
    """The store slab every chunk is a row range of (prefill_chunks), else None."""
    if not chunk_kvs or chunk_kvs[0].store is None:
        return None
    st = chunk_kvs[0].store
    return st if all(c.store is st for c in chunk_kvs) else None


def _select_from_store(weights, chunk_kvs, chunks, prompt_token_ids, config: SelectionConfig, timer: StageTimer):
    """assemble + attention-norm selection when the chunks live in one store
    slab: the query slab is gathered with every key rotated to its global
    position in ONE pass (the decode layout the recompute needs: no Kernel-1
    pass afterwards), on a second stream, while the scoring pass reads the
    chunk-local keys straight from the store (the rotation folded into its
    queries, exactly as on an assembled slab).  Same scores and selected set
    as assemble -> run_selection (the scorer sees identical operands)."""
    torch = E._torch()
    cfg = weights.config
    main = torch.cuda.current_stream()
    before = _after_previous(main)  # everything queued before this query
    cache = assemble_decode_layout(chunk_kvs, cfg.rope_base)  # enqueued on the current stream
    timer.mark("assemble")
    prompt = np.asarray(prompt_token_ids, dtype=np.int64)
    n = cache.context_length
    geometry = resolve_geometry(config, cache, int(prompt.size), cfg.max_position)
    assignment = assign_positions(geometry, chunks)
    nl = config.norm_layer if config.norm_layer is not None else default_norm_layer(cfg.n_layers)
    if not 0 <= nl < cfg.n_layers:
        from .errors import ConfigurationError

        raise ConfigurationError(f"norm_layer {nl} outside [0, {cfg.n_layers})")
    local = np.concatenate([c.prefill_positions for c in chunk_kvs])
    rows = np.concatenate([c.store_row0 + np.arange(c.length, dtype=np.int64) for c in chunk_kvs])
    group = E.PromptGroup(prompt, np.asarray(assignment.prompt_positions, np.int64),
                          E.segments_from_rows(rows, assignment.context_concat() - local))
    store_k, store_v = chunk_kvs[0].store
    overlap = STORE_OVERLAP
    hi = E._side_stream(2) if overlap else main
    if overlap:  # the scoring pass does not read the slab being gathered: no wait on it
        hi.wait_event(before)
    with torch.cuda.stream(hi):
        out = E.prompt_forward(weights, store_k, store_v, [group], capture_layer=nl)
        scores = out.scores.index_select(0, E.h2d(rows, store_k.device))  # store rows -> context order
        sel = SelectionResult(scores=scores, selected=select_topk(scores, config.resolve_budget(n)),
                              strategy=config.strategy.value, geometry=geometry.mode.value)
    if overlap:
        main.wait_stream(hi)
        for t in (scores, sel.selected):
            t.record_stream(main)
    return cache, sel


def assemble_select_recompute(weights, chunk_kvs: Sequence[ChunkKV], chunks: Sequence[ChunkSpec], prompt_token_ids,
                              selection: SelectionConfig, reorder: bool = False, chunk_score: str = "sum",
                              timer: Optional[StageTimer] = None) -> PathResult:
    timer = timer or StageTimer(enabled=False)
    timer.mark("start")
    rplan = None
    store = _shared_store(chunk_kvs)
    if (not reorder and store is not None and selection.strategy is Strategy.ATTENTION_NORM
            and weights.precision == "bf16"):
        cache, sel = _select_from_store(weights, chunk_kvs, chunks, prompt_token_ids, selection, timer)
        timer.mark("select")
    elif reorder:
        budget = selection.resolve_budget(sum(c.local_length for c in chunks))
        rplan, cache, sel = reorder_and_reselect(weights, chunks, prompt_token_ids, budget,
                                                 norm_layer=selection.norm_layer, chunk_score=chunk_score,
                                                 prefilled=chunk_kvs)
        timer.mark("reorder+select")
    else:
        cache = assemble(chunk_kvs)
        timer.mark("assemble")
        sel = run_selection(weights, chunks, cache, prompt_token_ids, selection)
        timer.mark("select")
    plan = make_plan(cache, sel.selected)
    cache = recompute_selected(weights, cache, plan)
    timer.mark("recompute")
    return PathResult(cache=cache, selection=sel, plan=plan, reorder=rplan)
