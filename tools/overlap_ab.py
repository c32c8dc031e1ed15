"""A/B of whole C2 queries as CUDA-graph replays (same process, same clocks):
the rotating gather serial before the scoring pass vs beside it on another
stream, with the gather's grid at several CTAs per SM (IFKV_GATHER_CPS; the
scoring kernels can only co-reside with a small gather grid).  Each variant
is its own QueryGraph (captured with its env), replays interleaved.
python tools/overlap_ab.py [--steps 8] [--variants serial:8,overlap:8,overlap:2,overlap:1]"""
import argparse
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_05353_b200 as P  # noqa: E402
from paper_2603_05353_b200 import pipeline as PL  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--variants", default="serial:8,overlap:8,overlap:2,overlap:1")
args = ap.parse_args()
cfg = P.llama3_8b_config()
w = P.DeviceWeights.random(cfg, seed=7)
task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=2048, prompt_length=32,
                       vocab_size=cfg.vocab_size)
g = P.generate_task(task, 0)
store = P.prefill_chunks(w, g.chunks)
sel = P.SelectionConfig(ratio=0.15)
graphs = {}
ref_sel = None
for v in args.variants.split(","):
    mode, cps = v.split(":")
    PL.STORE_OVERLAP = mode == "overlap"
    os.environ["IFKV_GATHER_CPS"] = cps
    qg = PL.QueryGraph(w, store, g.chunks, len(g.prompt_token_ids), sel)
    r = qg.run(g.prompt_token_ids)
    s = r.selection.selected_numpy().copy()
    if ref_sel is None:
        ref_sel, ref_k = s, r.cache.keys.float().sum().item()
    assert (s == ref_sel).all(), v
    kk = r.cache.keys.float().sum().item()
    print(f"{v}: selected set ok, keys checksum {'same' if kk == ref_k else f'DIFFERS {kk} vs {ref_k}'}", flush=True)
    graphs[v] = qg
res = {k: [] for k in graphs}
for it in range(args.steps + 2):
    order = list(graphs.items()) if it % 2 == 0 else list(reversed(graphs.items()))
    for name, qg in order:
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        qg.run(g.prompt_token_ids)
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            res[name].append(a.elapsed_time(b))
for k, v in res.items():
    print(f"{k:14s} median {statistics.median(v):7.2f} ms  min {min(v):7.2f}  all {' '.join(f'{x:.2f}' for x in v)}")
