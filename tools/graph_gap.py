import sys, time, statistics
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2603_05353_b200 as P
from paper_2603_05353_b200 import pipeline as PL
cfg = P.llama3_8b_config()
w = P.DeviceWeights.random(cfg, seed=7)
task = P.SyntheticTask(kind="uniform_noise", total_length=32768, fixed_size=2048, prompt_length=32, vocab_size=cfg.vocab_size)
g = P.generate_task(task, 0)
store = P.prefill_chunks(w, g.chunks)
sel = P.SelectionConfig(ratio=0.15)
qg = PL.query_graph(w, store, g.chunks, 32, sel)
for _ in range(3): qg.run(g.prompt_token_ids)
torch.cuda.synchronize()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): qg.graph.replay()
    b.record(); torch.cuda.synchronize()
    raw = a.elapsed_time(b) / 5
    a.record()
    for _ in range(5): qg.run(g.prompt_token_ids)
    b.record(); torch.cuda.synchronize()
    run = a.elapsed_time(b) / 5
    evs = []
    for _ in range(5):
        x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x.record(); qg.graph.replay(); y.record(); evs.append((x, y))
        torch.cuda.synchronize()
    single = statistics.median(x.elapsed_time(y) for x, y in evs)
    t0 = time.perf_counter(); qg.graph.replay(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"rep {rep}: back-to-back replay {raw:.2f} ms, run() loop {run:.2f} ms, single replay {single:.2f} ms, host launch {1e3*(t1-t0):.2f} ms", flush=True)
