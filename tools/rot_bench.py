"""A/B microbenchmark of Kernel 1 (in-place key re-rotation) at the C2 slab:
32 layers x 32768 rows x 8 kv heads x 128, rows of chunk 0 unmoved, 15 deltas.
Usage: python tools/rot_bench.py lib.so ..."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2603_05353_b200 import _native as N  # noqa: E402

_slab = {}


def run(lib, iters=10):
    N._lib = None
    N._fns.clear()
    N.load(Path(lib))
    from paper_2603_05353_b200 import cache as C
    from paper_2603_05353_b200 import engine as E

    if "k" not in _slab:
        torch.manual_seed(0)
        _slab["k"] = torch.randn(32, 32768, 8, 128, device="cuda", dtype=torch.bfloat16)
        _slab["ref"] = _slab["k"].clone()
    k = _slab["k"]
    deltas = np.repeat(np.arange(16, dtype=np.int64) * 2048, 2048)  # chunk c moves by 2048 c
    tab, cs = C._delta_table(deltas, 128, 5e5, "cuda")
    ts = []
    for i in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        E.rotate_rows(k, k, tab, cs)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    # correctness: one more rotation of a fresh copy vs the out-of-place path
    k.copy_(_slab["ref"])
    E.rotate_rows(k, k, tab, cs)
    want = torch.empty_like(k)
    E.rotate_rows(_slab["ref"], want, tab, cs)  # out of place (vector kernel)
    same = bool(torch.equal(k, want))
    k.copy_(_slab["ref"])
    moved = 30720 * 32 * 8 * 128 * 2 * 2
    return ms, moved / ms / 1e6, same


if __name__ == "__main__":
    for rep in range(2):
        for lib in sys.argv[1:]:
            ms, gbs, same = run(lib)
            print(f"{lib}: {ms * 1e3:.0f} us  {gbs:.0f} GB/s  bit-identical to out-of-place: {same}", flush=True)
