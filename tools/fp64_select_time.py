"""Time the float64 scoring mode (exact.py) against the fp32-accurate scorer
at the C2 shape (Llama-3-8B, 32K context, norm layer 19): python tools/fp64_select_time.py"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_05353_b200 as P  # noqa: E402

cfg = P.llama3_8b_config()
w = P.DeviceWeights.random(cfg, seed=7)
task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=2048, prompt_length=32,
                       vocab_size=cfg.vocab_size)
g = P.generate_task(task, 0)
kvs = P.prefill_chunks(w, g.chunks)
cache = P.assemble(kvs)
for prec in ("fp32", "fp64", "fp32", "fp64"):
    sc = P.SelectionConfig(ratio=0.15, score_precision=prec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.run_selection(w, g.chunks, cache, g.prompt_token_ids, sc)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    if prec == "fp32":
        s32 = r.selected_numpy()
    else:
        s64 = r.selected_numpy()
        import numpy as np
        print(f"sets differ in {np.setxor1d(s32, s64).size // 2} pair(s)")
    print(f"{prec}: run_selection {dt:.1f} ms", flush=True)
