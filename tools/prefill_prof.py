"""Per-kernel GPU time of the batched chunk prefill vs the full prefill (C2 shape).
python tools/prefill_prof.py"""
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_05353_b200 as P  # noqa: E402

cfg = P.llama3_8b_config()
w = P.DeviceWeights.random(cfg, seed=7)
task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=2048, prompt_length=32,
                       vocab_size=cfg.vocab_size)
g = P.generate_task(task, 0)
toks = np.concatenate([c.token_ids for c in g.chunks])
for name, fn in (("prefill_chunks", lambda: P.prefill_chunks(w, g.chunks)), ("full_prefill", lambda: P.full_prefill(w, toks))):
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        out = fn()
        torch.cuda.synchronize()
    del out
    tot = defaultdict(lambda: [0.0, 0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name[:90]][0] += e.device_time_total / 1e3
            tot[e.name[:90]][1] += 1
    print(f"== {name}: {sum(v[0] for v in tot.values()):.1f} ms GPU")
    for k, (t, n) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:8]:
        print(f"  {t:8.2f} ms {n:5d}  {k}")
