"""A/B of whole C2 steps in one process (same clocks): the store path (one
rotating gather, scoring from the store) vs the two-pass path (assemble, then
Kernel 1 inside the recompute), alternated step by step.
python tools/path_ab.py [--steps 8]"""
import argparse
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_05353_b200 as P  # noqa: E402
from paper_2603_05353_b200 import pipeline as PL  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=8)
args = ap.parse_args()
cfg = P.llama3_8b_config()
w = P.DeviceWeights.random(cfg, seed=7)
task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=2048, prompt_length=32,
                       vocab_size=cfg.vocab_size)
g = P.generate_task(task, 0)
store = P.prefill_chunks(w, g.chunks)
plain = [P.ChunkKV(c.chunk_id, c.token_ids, c.keys.clone(), c.values.clone(), c.prefill_positions, c.provenance,
                   c.model_fingerprint) for c in store]
sel = P.SelectionConfig(ratio=0.15)
variants = {"store+overlap": (store, True), "store serial": (store, False), "two-pass": (plain, True)}
res = {k: [] for k in variants}
for it in range(args.steps + 2):
    for name, (kvs, ov) in (variants.items() if it % 2 == 0 else reversed(list(variants.items()))):
        PL.STORE_OVERLAP = ov
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = P.assemble_select_recompute(w, kvs, g.chunks, g.prompt_token_ids, sel)
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            res[name].append(a.elapsed_time(b))
        del r
for k, v in res.items():
    print(f"{k:14s} median {statistics.median(v):7.2f} ms  min {min(v):7.2f}")
