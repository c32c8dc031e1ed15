"""Why the sharded bench's back-to-back device-timed steps are slower than
its per-step e2e: time the one-rank sharded step (a) back to back, (b) with a
device sync between steps, (c) back to back with the NVML clock sampler.
Usage: IFKV_FORCE_SHARDED=1 torchrun --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 tools/sharded_timing.py"""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2603_05353_b200 as P  # noqa: E402
from paper_2603_05353_b200 import sharding as SH  # noqa: E402

sys.argv = sys.argv[:1]
args = bench.parse()
world, rank, local = bench.dist_setup()
comm = SH.TorchComm()
cfg = bench.model_config(args)
weights = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
gen = P.generate_task(bench.make_task(args, cfg), seed=0)
chunks, prompt = gen.chunks, gen.prompt_token_ids
shard = SH.make_shard([c.local_length for c in chunks], rank, world)
my_kvs = [P.prefill_chunk(weights, chunks[c]) for c in shard.chunk_ids]
sel_cfg = P.SelectionConfig(ratio=args.ratio)


def step():
    local_cache = P.assemble(my_kvs)
    res = SH.sharded_select(weights, shard, local_cache, prompt, sel_cfg, comm)
    SH.sharded_recompute(weights, shard, local_cache, res.selected, comm)
    return res


for _ in range(3):
    step()
torch.cuda.synchronize()


def timed(n, sync_between, sampler=False):
    cs = None
    if sampler:
        cs = bench.ClockSampler(torch.cuda.current_device())
        cs.start()
        cs.begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        step()
        if sync_between:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / n
    if cs:
        cs.stop()
    return e0.elapsed_time(e1) / n, wall


for name, kw in [("back-to-back", dict(sync_between=False)), ("sync between", dict(sync_between=True)),
                 ("back-to-back + sampler", dict(sync_between=False, sampler=True)),
                 ("back-to-back again", dict(sync_between=False))]:
    ev, wall = timed(3, **kw)
    print(f"{name:26s} events {ev:8.2f} ms/step, wall {wall:8.2f} ms/step", flush=True)
