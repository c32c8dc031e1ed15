"""In-tree build of the sm_100a native library ``_build/libifkv.so``.

Every ``csrc/*.cu`` is compiled with nvcc for ``sm_100a`` only
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``) and linked into one
shared library exporting the C ABI declared in ``include/ifkv.h``.  The
library lives inside the package directory so that it travels with the repo
snapshot to the GPU box (a JIT cache would not).
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_build"
LIB = OUT_DIR / "libifkv.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
    "-Xptxas",
    "-v",
    f"-I{INCLUDE}",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build the ifkv native library")


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _digest(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, out_dir: Path = OUT_DIR, extra_flags=()) -> Path:
    """Compile all kernels; skip when sources and flags are unchanged.
    ``out_dir`` / ``extra_flags`` build kernel variants for A/B timing."""
    out_dir = Path(out_dir)
    lib = out_dir / "libifkv.so"
    deps = list(_sources()) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    stamp = out_dir / "libifkv.sha256"
    digest = _digest(deps) + " ".join(extra_flags)
    if not force and lib.exists() and stamp.exists() and stamp.read_text() == digest:
        return lib
    out_dir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    objs = []

    def compile_one(src: Path):
        obj = out_dir / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra_flags, "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
        (out_dir / (src.stem + ".ptxas.txt")).write_text(res.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, _sources()))
    cmd = [nvcc, *ARCH, "-shared", "-o", str(lib), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    stamp.write_text(digest)
    if verbose:
        print(f"built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
