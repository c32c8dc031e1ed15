"""IFKC chunk-cache files <-> HBM (reference cache.py:103-199, README.md:170-182).

Byte-compatible with the reference container: magic "IFKC", version u32 = 1,
model fingerprint u64, chunk id (u32 length + utf-8), length / n_layers /
n_heads / d_head as u32, provenance u8, precision code u8, token ids and
prefill positions as i64, then per layer K then V as raw little-endian
floats, then a u64 blake2b-8 checksum of every preceding byte.  Precision
codes 0 = f32 and 1 = f64 are the reference's; this package adds 2 = bf16
(raw bfloat16 bits), the HBM-native precision, so a prepared context loads
with one host->device copy per tensor and no conversion.

Loading stages the payload in pinned host memory and copies it to the
device; K and V of all layers land in the [L, len, Hkv, Dh] layout the
assembler gathers from.
"""

from __future__ import annotations

import hashlib
import struct
from pathlib import Path

import numpy as np

from .cache import ChunkKV, Provenance
from .errors import ConfigurationError, DataFormatError

MAGIC = b"IFKC"
VERSION = 1
CODE_F32, CODE_F64, CODE_BF16 = 0, 1, 2
_ITEM = {CODE_F32: 4, CODE_F64: 8, CODE_BF16: 2}


def _hash64(data) -> int:
    return int.from_bytes(hashlib.blake2b(data, digest_size=8).digest(), "little")


def _code_of(dtype) -> int:
    import torch

    if dtype == torch.float32:
        return CODE_F32
    if dtype == torch.float64:
        return CODE_F64
    if dtype == torch.bfloat16:
        return CODE_BF16
    raise ConfigurationError(f"unsupported cache dtype {dtype}")


def save_cache(cache: ChunkKV, path) -> None:
    """Write a device ChunkKV as an IFKC file (cache.py:110-140)."""
    import torch

    L, n, hkv, dh = cache.keys.shape
    code = _code_of(cache.keys.dtype)
    buf = bytearray()
    buf += MAGIC
    buf += struct.pack("<I", VERSION)
    buf += struct.pack("<Q", cache.model_fingerprint & 0xFFFFFFFFFFFFFFFF)
    cid = cache.chunk_id.encode()
    buf += struct.pack("<I", len(cid)) + cid
    buf += struct.pack("<IIII", n, L, hkv, dh)
    buf += struct.pack("<BB", int(cache.provenance), code)
    buf += np.ascontiguousarray(cache.token_ids, dtype="<i8").tobytes()
    buf += np.ascontiguousarray(cache.prefill_positions, dtype="<i8").tobytes()
    kv = torch.stack([cache.keys, cache.values], dim=1).contiguous().cpu()  # [L, 2, n, Hkv, Dh]
    raw = kv.view(torch.int16).numpy() if code == CODE_BF16 else kv.numpy()
    buf += raw.astype(raw.dtype.newbyteorder("<"), copy=False).tobytes()
    buf += struct.pack("<Q", _hash64(bytes(buf)))
    Path(path).write_bytes(bytes(buf))


def load_cache(path, device="cuda", dtype=None) -> ChunkKV:
    """Read an IFKC file into HBM (cache.py:143-199).  ``dtype`` (torch)
    converts on the device; default keeps the file precision."""
    import torch

    data = Path(path).read_bytes()
    if len(data) < 8 or data[:4] != MAGIC:
        raise DataFormatError("bad magic: not an IFKC cache file")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != VERSION:
        raise DataFormatError(f"unsupported cache version {version}, expected {VERSION}")
    if len(data) < 16:
        raise DataFormatError("truncated cache file")
    payload = memoryview(data)[:-8]
    (stored,) = struct.unpack("<Q", data[-8:])
    if _hash64(payload) != stored:
        raise DataFormatError("cache checksum mismatch (corrupt file)")
    off = 8
    (fp,) = struct.unpack_from("<Q", data, off)
    off += 8
    (cl,) = struct.unpack_from("<I", data, off)
    off += 4
    if off + cl > len(payload):
        raise DataFormatError("truncated cache file")
    cid = bytes(data[off:off + cl]).decode()
    off += cl
    if off + 18 > len(payload):
        raise DataFormatError("truncated cache file")
    n, L, hkv, dh = struct.unpack_from("<IIII", data, off)
    off += 16
    prov, code = struct.unpack_from("<BB", data, off)
    off += 2
    if code not in _ITEM:
        raise DataFormatError(f"unknown precision code {code}")
    need = off + 16 * n + 2 * L * n * hkv * dh * _ITEM[code]
    if need > len(payload):
        raise DataFormatError("truncated cache file")
    if need != len(payload):
        raise DataFormatError("trailing bytes inside cache payload")
    tok = np.frombuffer(data, dtype="<i8", count=n, offset=off).astype(np.int64)
    off += 8 * n
    pos = np.frombuffer(data, dtype="<i8", count=n, offset=off).astype(np.int64)
    off += 8 * n
    count = 2 * L * n * hkv * dh
    np_dt = {CODE_F32: "<f4", CODE_F64: "<f8", CODE_BF16: "<i2"}[code]
    raw = np.frombuffer(data, dtype=np_dt, count=count, offset=off).reshape(L, 2, n, hkv, dh)
    host = torch.from_numpy(raw.copy())
    if code == CODE_BF16:
        host = host.view(torch.bfloat16)
    host = host.pin_memory() if torch.cuda.is_available() and str(device).startswith("cuda") else host
    dev = host.to(device, non_blocking=True)
    if dtype is not None:
        dev = dev.to(dtype)
    try:
        provenance = Provenance(prov)
    except ValueError as exc:
        raise DataFormatError(f"unknown provenance code {prov}") from exc
    return ChunkKV(cid, tok, dev[:, 0], dev[:, 1], pos, provenance, fp)
