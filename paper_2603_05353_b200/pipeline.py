"""The timed path as one call: assemble -> (reorder) -> select -> recompute
(reference harness.py:433-456 minus chunk prefill and decode, which sit
outside the metric: prepared context, time to the recomputed cache).

``assemble_select_recompute`` is the public entry point the benchmark's
end-to-end leg calls; ``StageTimer`` records CUDA events between stages on
the current stream.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from .cache import AssembledCache, ChunkKV, assemble
from .positions import ChunkSpec
from .recompute import RecomputePlan, make_plan, recompute_selected
from .reorder import ReorderPlan, reorder_and_reselect
from .selection import SelectionConfig, SelectionResult, run_selection


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


def assemble_select_recompute(weights, chunk_kvs: Sequence[ChunkKV], chunks: Sequence[ChunkSpec], prompt_token_ids,
                              selection: SelectionConfig, reorder: bool = False, chunk_score: str = "sum",
                              timer: Optional[StageTimer] = None) -> PathResult:
    timer = timer or StageTimer(enabled=False)
    timer.mark("start")
    rplan = None
    if reorder:
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
