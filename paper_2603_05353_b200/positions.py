"""RoPE position geometries for chunked contexts (reference positions.py:1-168).

Host-side integer logic: it decides, per chunk, the rotation delta the
kernels fold into the keys (Kernel 1) or into the queries (scorer).

  GLOBAL  chunks at their concatenated offsets, prompt right after them;
  HL-HP   chunks at local positions, prompt after the longest chunk;
  HL-TP   chunks at local positions, prompt at its original global index;
  TL-TP   chunks packed so the context ends one position before the prompt.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Optional, Sequence

import numpy as np

from .errors import ConfigurationError


class GeometryMode(Enum):
    GLOBAL = "GLOBAL"
    HL_HP = "HL-HP"
    HL_TP = "HL-TP"
    TL_TP = "TL-TP"

    @classmethod
    def parse(cls, name) -> "GeometryMode":
        """Case-insensitive; '-' and '_' are interchangeable (positions.py:38-48)."""
        if isinstance(name, cls):
            return name
        wanted = str(name).strip().upper().replace("_", "-")
        for mode in cls:
            if mode.value == wanted:
                return mode
        raise ConfigurationError(
            f"unknown geometry mode {name!r}; expected one of {', '.join(m.value for m in cls)}")


@dataclass
class ChunkSpec:
    """A context chunk: id, token ids and declared position (positions.py:51-64)."""

    chunk_id: str
    token_ids: np.ndarray
    declared_order_index: int = 0
    local_length: int = field(init=False)

    def __post_init__(self):
        self.token_ids = np.asarray(self.token_ids, dtype=np.int64)
        if self.token_ids.ndim != 1:
            raise ConfigurationError(f"chunk {self.chunk_id!r} token_ids must be 1-D")
        self.local_length = int(self.token_ids.size)


@dataclass
class GeometryConfig:
    """One layout of (chunks, prompt) (positions.py:67-97).  prompt_offset is
    the prompt's original global index (default: sum of chunk lengths); HL-TP
    starts the prompt there and TL-TP packs the chunks against it."""

    mode: GeometryMode
    prompt_length: int
    chunk_lengths: tuple
    prompt_offset: Optional[int] = None
    max_position: Optional[int] = None

    def __post_init__(self):
        self.mode = GeometryMode.parse(self.mode)
        self.chunk_lengths = tuple(int(n) for n in self.chunk_lengths)
        if any(n < 1 for n in self.chunk_lengths):
            raise ConfigurationError("chunk lengths must all be >= 1")
        if self.prompt_length < 0:
            raise ConfigurationError("prompt_length must be >= 0")
        if self.prompt_offset is not None and self.prompt_offset < 0:
            raise ConfigurationError("prompt_offset must be >= 0")

    @property
    def context_length(self) -> int:
        return sum(self.chunk_lengths)


@dataclass
class PositionAssignment:
    context_positions: list  # per chunk, consecutive increasing int64
    prompt_positions: np.ndarray

    def context_concat(self) -> np.ndarray:
        if not self.context_positions:
            return np.zeros(0, dtype=np.int64)
        return np.concatenate(self.context_positions)

    def chunk_starts(self) -> np.ndarray:
        """First position of every chunk (chunks are runs of consecutive positions)."""
        return np.array([int(p[0]) for p in self.context_positions], dtype=np.int64)


def _chunk_starts(mode: GeometryMode, lengths, anchor: int):
    if mode is GeometryMode.GLOBAL:
        return np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64), int(sum(lengths))
    if mode is GeometryMode.HL_HP:
        return np.zeros(len(lengths), np.int64), int(max(lengths))
    if mode is GeometryMode.HL_TP:
        return np.zeros(len(lengths), np.int64), anchor
    tail = np.cumsum(np.asarray(lengths)[::-1])[::-1]  # TL-TP: suffix sums
    starts = anchor - tail
    if starts[0] < 0:
        raise ConfigurationError(
            f"TL-TP pack underflows: prompt offset {anchor} is smaller than the total context length {sum(lengths)}")
    return starts.astype(np.int64), anchor


def assign_positions(config: GeometryConfig, chunks: Sequence[ChunkSpec]) -> PositionAssignment:
    """Positions of every context and prompt token (positions.py:111-168)."""
    lengths = config.chunk_lengths
    if len(chunks) != len(lengths):
        raise ConfigurationError(f"{len(chunks)} chunks supplied for {len(lengths)} declared lengths")
    for c, n in zip(chunks, lengths):
        if c.local_length != n:
            raise ConfigurationError(f"chunk {c.chunk_id!r} has length {c.local_length}, declared {n}")
    total = sum(lengths)
    anchor = total if config.prompt_offset is None else int(config.prompt_offset)
    if lengths:
        starts, p0 = _chunk_starts(config.mode, lengths, anchor)
    else:
        starts, p0 = np.zeros(0, np.int64), (anchor if config.mode in (GeometryMode.HL_TP, GeometryMode.TL_TP) else 0)
    ctx = [int(s) + np.arange(n, dtype=np.int64) for s, n in zip(starts, lengths)]
    prompt = int(p0) + np.arange(config.prompt_length, dtype=np.int64)
    if config.max_position is not None:
        tops = [int(c[-1]) for c in ctx] + ([int(prompt[-1])] if prompt.size else [0])
        top = max(tops)
        if top >= config.max_position:
            raise ConfigurationError(f"assigned position {top} overflows max_position {config.max_position}")
    return PositionAssignment(context_positions=ctx, prompt_positions=prompt)
