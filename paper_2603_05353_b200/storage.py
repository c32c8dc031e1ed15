"""IFKC chunk-cache files <-> HBM (reference cache.py:103-199, README.md:170-182).

The reference container: magic "IFKC", version u32 = 1, model fingerprint
u64, chunk id (u32 length + utf-8), length / n_layers / n_heads / d_head as
u32, provenance u8, precision code u8, token ids and prefill positions as
i64, then per layer K then V as raw little-endian floats, then a u64
blake2b-8 checksum of every preceding byte.  Precision codes 0 = f32 and
1 = f64 are the reference's; this package adds 2 = bf16 (raw bfloat16 bits),
the HBM-native precision.  Files with codes 0/1 are byte-compatible both
ways; the reference's load_cache rejects code 2, so ``save_cache`` writes a
bf16 cache as f32 (an exact upcast) unless ``precision="bf16"`` asks for the
compact native file.

Loading reads the file once, straight into pinned host memory, checks the
checksum there and copies the K/V payload to the device with one
asynchronous copy (no intermediate host copy); ``load_caches`` overlaps the
read of the next file with the copy of the previous one.  K and V of all
layers land in the [L, len, Hkv, Dh] layout the assembler gathers from;
``dtype`` converts on the device.
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


def save_cache(cache: ChunkKV, path, precision=None) -> None:
    """Write a ChunkKV as an IFKC file (cache.py:110-140).  ``precision``:
    "f32", "f64", "bf16" or None (the tensors' own precision, except that
    bf16 tensors are written as exact f32 so the reference can read them)."""
    import torch

    L, n, hkv, dh = cache.keys.shape
    want = {None: None, "f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}
    if precision not in want:
        raise ConfigurationError(f"unknown cache precision {precision!r}, expected f32, f64 or bf16")
    dt = want[precision] or (torch.float32 if cache.keys.dtype == torch.bfloat16 else cache.keys.dtype)
    if dt != cache.keys.dtype:
        cache = ChunkKV(cache.chunk_id, cache.token_ids, cache.keys.to(dt), cache.values.to(dt),
                        cache.prefill_positions, cache.provenance, cache.model_fingerprint)
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


def _read_pinned(path, pin: bool):
    """The whole file in one (pinned) host buffer: torch uint8 tensor."""
    import torch

    p = Path(path)
    size = p.stat().st_size
    buf = torch.empty(size, dtype=torch.uint8, pin_memory=pin)
    with open(p, "rb", buffering=0) as f:
        got = f.readinto(memoryview(buf.numpy()))
    if got != size:
        raise DataFormatError("truncated cache file (short read)")
    return buf


def load_cache(path, device="cuda", dtype=None) -> ChunkKV:
    """Read an IFKC file into HBM (cache.py:143-199).  ``dtype`` (torch)
    converts on the device; default keeps the file precision."""
    import torch

    pin = torch.cuda.is_available() and str(device).startswith("cuda")
    buf = _read_pinned(path, pin)
    data = memoryview(buf.numpy())
    if len(data) < 8 or bytes(data[:4]) != MAGIC:
        raise DataFormatError("bad magic: not an IFKC cache file")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != VERSION:
        raise DataFormatError(f"unsupported cache version {version}, expected {VERSION}")
    if len(data) < 16:
        raise DataFormatError("truncated cache file")
    payload = data[:-8]
    (stored,) = struct.unpack_from("<Q", data, len(data) - 8)
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
    arr = buf.numpy()
    tok = np.frombuffer(arr, dtype="<i8", count=n, offset=off).astype(np.int64)
    off += 8 * n
    pos = np.frombuffer(arr, dtype="<i8", count=n, offset=off).astype(np.int64)
    off += 8 * n
    try:
        provenance = Provenance(prov)
    except ValueError as exc:
        raise DataFormatError(f"unknown provenance code {prov}") from exc
    # K/V payload: one async copy of the raw bytes from the pinned buffer, typed
    # on the device (the device allocation is aligned, the file offset need not be)
    nbytes = 2 * L * n * hkv * dh * _ITEM[code]
    raw = buf[off:off + nbytes]
    dev = raw.to(device, non_blocking=True) if pin else raw.clone()
    tdt = {CODE_F32: torch.float32, CODE_F64: torch.float64, CODE_BF16: torch.bfloat16}[code]
    kv = dev.view(tdt).view(L, 2, n, hkv, dh)
    if dtype is not None and dtype != tdt:
        kv = kv.to(dtype)
    return ChunkKV(cid, tok, kv[:, 0], kv[:, 1], pos, provenance, fp)


def load_caches(paths, device="cuda", dtype=None):
    """Load several IFKC files; the host read + checksum of file i+1 overlaps
    the asynchronous host->device copy of file i."""
    return [load_cache(p, device=device, dtype=dtype) for p in paths]
