"""Synthetic inputs: the reference harness's task generator (harness.py:180-295).

Random weights make QA accuracy meaningless; the benchmark and the parity
tests use the reference's synthetic contexts, drawn with the same PCG64
stream so token ids are identical to the reference's for the same seed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from .errors import ConfigurationError
from .positions import ChunkSpec

RESERVED_BAND = 64  # needle / prompt ids live in the top band (harness.py:79)
FIRST_NOISE_ID = 2


@dataclass
class SyntheticTask:
    kind: str = "needle"  # "needle" | "uniform_noise"
    total_length: int = 256
    needle_depth: Optional[float] = None
    depth_range: Tuple[float, float] = (0.0, 1.0)
    fixed_size: Optional[int] = 64
    boundaries: Optional[tuple] = None
    prompt_length: int = 8
    prompt_needle_copies: int = 1
    vocab_size: int = 256

    def __post_init__(self):
        if self.kind not in ("needle", "uniform_noise"):
            raise ConfigurationError(f"unknown task kind {self.kind!r}")
        if self.total_length < 1 or self.prompt_length < 1:
            raise ConfigurationError("total_length and prompt_length must be >= 1")
        if (self.fixed_size is None) == (self.boundaries is None):
            raise ConfigurationError("exactly one of fixed_size or boundaries must be set")
        if self.fixed_size is not None and self.fixed_size < 1:
            raise ConfigurationError("fixed_size must be >= 1")
        if self.vocab_size < RESERVED_BAND + FIRST_NOISE_ID + 1:
            raise ConfigurationError(f"vocab_size too small, need > {RESERVED_BAND + FIRST_NOISE_ID}")
        if self.needle_depth is not None and self.needle_depth < 0:
            raise ConfigurationError("needle_depth must be >= 0")
        lo, hi = float(self.depth_range[0]), float(self.depth_range[1])
        if not 0.0 <= lo <= hi <= 1.0:
            raise ConfigurationError(f"depth_range must satisfy 0 <= lo <= hi <= 1, got {self.depth_range}")
        self.depth_range = (lo, hi)
        if not 1 <= self.prompt_needle_copies <= self.prompt_length:
            raise ConfigurationError("prompt_needle_copies must be in [1, prompt_length]")


@dataclass
class GeneratedTask:
    chunks: List[ChunkSpec]
    prompt_token_ids: np.ndarray
    needle_index: Optional[int]
    needle_token: Optional[int]
    task: SyntheticTask
    seed: int

    def chunk_lengths(self) -> tuple:
        return tuple(c.local_length for c in self.chunks)


def chunk_lengths_for(task: SyntheticTask) -> List[int]:
    n = task.total_length
    if task.fixed_size is not None:
        full, rest = divmod(n, task.fixed_size)
        return [task.fixed_size] * full + ([rest] if rest else [])
    cuts = sorted(int(b) for b in task.boundaries)
    if any(b <= 0 or b >= n for b in cuts) or len(set(cuts)) != len(cuts):
        raise ConfigurationError("passage boundaries must be distinct interior offsets")
    edges = [0] + cuts + [n]
    return [b - a for a, b in zip(edges[:-1], edges[1:])]


def generate_task(task: SyntheticTask, seed: int) -> GeneratedTask:
    """Same draws as harness.py:244-295: noise tokens, reserved-band
    permutation, optional needle depth, then the chunk split."""
    rng = np.random.default_rng(seed)
    band0 = task.vocab_size - RESERVED_BAND
    tokens = rng.integers(FIRST_NOISE_ID, band0, size=task.total_length, dtype=np.int64)
    band = rng.permutation(np.arange(band0, task.vocab_size, dtype=np.int64))
    needle_index = needle_token = None
    if task.kind == "needle":
        needle_token = int(band[0])
        depth = task.needle_depth if task.needle_depth is not None else float(
            rng.uniform(task.depth_range[0], task.depth_range[1]))
        needle_index = int(math.floor(depth * task.total_length))
        if needle_index >= task.total_length:
            raise ConfigurationError(f"needle depth {depth} places the needle beyond the context")
        tokens[needle_index] = needle_token
        copies = task.prompt_needle_copies
        prompt = np.concatenate([[needle_token] * copies, band[1:task.prompt_length - copies + 1]]).astype(np.int64)
    else:
        prompt = band[:task.prompt_length].astype(np.int64)
    if prompt.size < task.prompt_length:
        raise ConfigurationError("prompt_length exceeds the reserved token band")
    chunks, start = [], 0
    for ci, n in enumerate(chunk_lengths_for(task)):
        chunks.append(ChunkSpec(chunk_id=f"c{ci}", token_ids=tokens[start:start + n], declared_order_index=ci))
        start += n
    return GeneratedTask(chunks, prompt, needle_index, needle_token, task, seed)


def make_chunks(token_ids, lengths) -> List[ChunkSpec]:
    """Split a token array into ChunkSpecs of the given lengths."""
    out, start = [], 0
    for i, n in enumerate(lengths):
        out.append(ChunkSpec(chunk_id=f"c{i}", token_ids=np.asarray(token_ids)[start:start + n],
                             declared_order_index=i))
        start += n
    if start != len(token_ids):
        raise ConfigurationError("chunk lengths do not cover the token array")
    return out
