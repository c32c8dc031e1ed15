"""ctypes binding of the sm_100a native library (C ABI in include/ifkv.h).

There is no fallback: if ``_build/libifkv.so`` is missing or no CUDA device
is present, every compute entry point raises NativeError.  Status codes map
to the package's exceptions: IFKV_ERR_ARG -> ConfigurationError,
IFKV_ERR_CUDA -> NativeError, each with the library's thread-local message.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ConfigurationError, NativeError

# IFKV_LIB: load an A/B build (tools/build_variants.py -> _ab/<name>/libifkv.so) instead
LIB_PATH = Path(os.environ.get("IFKV_LIB", Path(__file__).resolve().parent / "_build" / "libifkv.so"))

IFKV_F32, IFKV_BF16 = 0, 1
OUT_F32, OUT_BF16, OUT_SPLIT3 = 0, 1, 2
AGG_NONE, AGG_SUM, AGG_MEAN, AGG_MAX = -1, 0, 1, 2
AGG_CODES = {"sum": AGG_SUM, "mean": AGG_MEAN, "max": AGG_MAX}

P, I32, I64, F32, F64 = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double

# name -> argtypes (restype is always c_int status unless noted)
SIGNATURES = {
    "ifkv_rope_table": [P, I32, I32, F64, P, P],
    "ifkv_rotate_rows": [I32, P, P, I64, I32, I32, I32, I32, P, P, P],
    "ifkv_assemble_gather": [I32, I32, P, P, P, P, P, P, P, I64, I32, I32, P],
    "ifkv_assemble_gather_rotate": [I32, I32, P, P, P, P, P, P, P, I32, P, P, I64, I32, I32, P],
    "ifkv_add_rmsnorm": [P, P, I32, I32, P, I32, I32, I32, P, P],
    "ifkv_silu_mul": [P, I32, I32, I32, I32, I32, I32, P, P],
    "ifkv_embed_rows": [P, I32, P, I32, I32, P, P],
    "ifkv_split3": [P, I64, P, P],
    "ifkv_row_dist_accum": [P, P, I32, I32, P, P],
    "ifkv_prompt_mm": [P, I32, I32, I32, P, I32, I32, P, P],
    "ifkv_qkv_rope_scatter": [P, I32, I32, I32, I32, I32, I32, P, I32, P, P, P, P, P],
    "ifkv_prompt_attn_partial": [I32, P, P, P, P, P, P, I32, I32, I32, I32, I32, I32, F32, P, P, P],
    "ifkv_prompt_attn_merge": [P, P, P, I32, I32, I32, I32, I32, I32, P, P, P, P],
    "ifkv_prompt_attn_merge_rows": [P, P, P, I32, I32, I32, I32, I32, I32, P, P, P, P],
    "ifkv_prompt_attn_tc_supported": [I32, I32, I32, I32, I32],
    "ifkv_prompt_attn_partial_tc": [P, I32, P, P, I32, P, I32, I32, I32, I32, I32, F32, P, P, P],
    "ifkv_score_columns_tc": [P, I32, P, I32, P, I32, I32, P, I32, I32, I32, F32, P, P, P],
    "ifkv_score_columns": [I32, P, P, P, I32, P, I32, I32, I32, I32, F32, P, P],
    "ifkv_rotate_queries": [P, I32, I32, I32, I32, P, P, I32, P, P, P, P],
    "ifkv_topk_segments": [P, P, P, P, I32, P, I32, P, P],
    "ifkv_recompute_attn": [I32, P, P, P, P, I32, I32, I32, I32, I32, F32, P, P],
    "ifkv_recompute_attn_range": [I32, P, P, P, P, P, I32, I32, I32, I32, I32, F32, P, P],
    "ifkv_recompute_attn_simt": [I32, P, P, P, P, I32, I32, I32, I32, I32, F32, P, P],
    "ifkv_recompute_attn_tc_supported": [I32, I32, I32, I32],
    "ifkv_recompute_attn_partial": [I32, P, P, P, P, I32, I32, I32, I32, I32, F32, P, P, P],
    "ifkv_merge_partials": [P, P, I32, I64, I32, P, P, P],
    "ifkv_merge_prompt_states": [P, P, I32, I32, I32, I32, I32, P, P, P],
    "ifkv_prompt_qkv": [P, I32, I32, I32, I32, I32, I32, P, P, P, P, I32, P, P, P, P, P, P],
    "ifkv_gemm": [P, I64, I32, I32, P, I32, I32, P, I64, I32, I32, P],
    "ifkv_gemm_qkv_rope_scatter": [P, I64, I32, I32, P, I32, I32, I32, P, P, P, P, P, I32, P],
    "ifkv_gemm_swiglu": [P, I64, I32, I32, P, I32, P, I32, P],
}
EXPORTS = tuple(SIGNATURES) + ("ifkv_last_error", "ifkv_abi_version")

_lock = threading.Lock()
_lib = None


def load(path: Path = LIB_PATH):
    """Load (once) and type the library; raise NativeError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not path.exists():
            raise NativeError(
                f"native library {path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(str(path))
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.ifkv_last_error.argtypes = []
        lib.ifkv_last_error.restype = C.c_char_p
        lib.ifkv_abi_version.argtypes = []
        lib.ifkv_abi_version.restype = C.c_int
        _fns.clear()
        _lib = lib
        return lib


LAUNCH_COUNT = [0]  # entry-point calls that enqueue kernels (bench gpu_launches)


_fns: dict = {}


def call(name: str, *args) -> int:
    """Invoke an entry point and translate its status code."""
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(load(), name)
    query = name.endswith("_supported")
    if not query:
        LAUNCH_COUNT[0] += 1
    status = fn(*args)
    if status == 0 or query:
        return status
    lib = load()
    msg = lib.ifkv_last_error().decode(errors="replace")
    if status == 2:
        raise ConfigurationError(f"{name}: {msg}")
    raise NativeError(f"{name}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


_stream_fn = None


def stream_handle() -> int:
    """The current CUDA stream of the current device (raw cudaStream_t).
    Uses torch's direct C accessors when present: torch.cuda.current_stream()
    costs several microseconds of Python per call (device-index resolution,
    availability checks) and the scoring pass makes ~12 entry-point calls
    per layer, so on a synchronous query it was a visible share of the host
    time that paces the GPU."""
    global _stream_fn
    if _stream_fn is None:
        import torch

        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        dev = getattr(torch._C, "_cuda_getDevice", None)
        if raw is not None and dev is not None:
            _stream_fn = lambda: raw(dev())  # noqa: E731
        else:  # pragma: no cover - older torch
            _stream_fn = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    return _stream_fn()
