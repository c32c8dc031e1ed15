"""The path's immediate consumer: the prompt forward over the decode view and
the first generated token (reference harness.py:458-469: decode_view, then
``forward(prompt at positions n..n+m-1, injected=decode view)``, greedy argmax
of the last position's logits, model.py:465-467).

The decode view is never materialised: each constant-delta run of cached keys
is read through the rotated prompt queries (q . R(d) k == (R(-d) q) . k), so
this works on any cache -- freshly assembled (chunk-local rotations) or after
``recompute_selected`` (already in the decode layout, delta 0 everywhere).
fp32-accurate like the scorer (3-term bf16 operand splits in bf16 mode).
"""

from __future__ import annotations

import numpy as np

from . import engine as E
from .cache import AssembledCache, decode_targets
from .errors import ConfigurationError


def first_token_logits(weights, cache: AssembledCache, prompt_token_ids):
    """fp32 logits [vocab] of the last prompt position over the cache's
    context rows in the global decode layout."""
    cfg = weights.config
    prompt = np.asarray(prompt_token_ids, dtype=np.int64)
    if prompt.ndim != 1 or prompt.size == 0:
        raise ConfigurationError("token_ids must be a nonempty 1-D sequence")
    if prompt.min() < 0 or prompt.max() >= cfg.vocab_size:
        raise ConfigurationError("token id outside vocabulary")
    n = cache.context_length
    deltas = decode_targets(cache)[:n] - cache.row_positions[:n]
    group = E.PromptGroup(prompt, n + np.arange(prompt.size, dtype=np.int64), E.segments_from_deltas(deltas))
    return E.prompt_forward(weights, cache.keys, cache.values, [group], want_logits=True).logits[0]


def greedy_token(logits) -> int:
    """Greedy argmax, lowest id on ties (model.py:465-467)."""
    import torch

    if isinstance(logits, torch.Tensor):
        return int(torch.argmax(logits).item())  # torch.argmax returns the first maximal index
    return int(np.argmax(logits))
