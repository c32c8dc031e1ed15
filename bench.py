"""Benchmark: InfoFlow-KV query-time context assembly on B200.

Metric (BASELINE.json): assemble + select + recompute time and ctx tok/s for
a Llama-3-8B-shaped model (random-init bf16 weights), a 32K-token context of
16 x 2048 chunks (synthetic uniform-noise tokens from the reference's task
generator) and a 15% recompute ratio, on one B200.  A step = one pass of the
path over the prepared (HBM-resident) chunk KVs: assemble -> attention-norm
selection (fp32-accurate prompt forward to layer 19 + exact top-k) ->
selective recompute of 4916 tokens through 32 layers with in-place K/V
scatter.  value = context tokens / step time, summed over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the ranks chunk-shard ONE context (zig-zag chunk
ownership, NCCL softmax-state merges, top-k candidate all-gather, sparse-query
partial attention).  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = {"hbm_gbs": 6534.1, "bf16_tflops": 1659.4, "bf16_tflops_sustained": 1395.0, "source": "fallback"}
try:
    _p = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    PEAKS.update({k: _p[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in _p})
    PEAKS["source"] = "measured (MEASURED_PEAKS.json)"
except Exception:
    pass

HBM_SPEC_GBS = 8000.0  # the B200 HBM3e spec figure the north star cites (~8 TB/s)
METRIC = "assemble+select+recompute ms & ctx tok/s, Llama-3-8B shape, 32K ctx, 15% recompute"

# DRAM bytes per launch of the roofline kernels from one `ncu --set full`
# capture (tools/gpu_prof.sh -> tools/ncu_traffic.py), committed under profiles/.
TRAFFIC_FILE = ROOT / "profiles" / "r2_ncu_traffic.json"


def ncu_traffic(name):
    try:
        t = json.loads(TRAFFIC_FILE.read_text())[name]
        return t["dram_read_bytes"] + t["dram_write_bytes"]
    except Exception:
        return None


# Max elementwise relative error of the fp32-accurate scores against the
# float64 oracle, measured at Llama-3-8B width over the same 32K context
# (tests/test_gpu_headline.py, 4 layers: 4.35e-6; Qwen2.5-VL width 1.56e-6).
SCORE_REL_ERR = 4.35e-6


def boundary_margin(scores, k):
    """SURVEY §7 hard part 1: the score gap at the selection boundary (k-th vs
    (k+1)-th best) relative to the k-th score, divided by the largest score
    movement the measured error allows (both scores moving toward each other).
    > 1: the selected set is certified by the error bound; <= 1: it matches
    the oracle only if the boundary tokens' actual errors are smaller."""
    s = np.sort(np.asarray(scores, np.float64))[::-1]
    if k <= 0 or k >= s.size:
        return None
    gap = (s[k - 1] - s[k]) / s[k - 1]
    return {"gap_rel": gap, "score_rel_err_bound": SCORE_REL_ERR, "margin": gap / (2 * SCORE_REL_ERR),
            "err_source": "tests/test_gpu_headline.py (C2 width, 4 layers, vs float64 oracle)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--chunk", type=int, default=2048)
    ap.add_argument("--ratio", type=float, default=0.15)
    ap.add_argument("--layers", type=int, default=0, help="override model depth (debug only)")
    ap.add_argument("--model", choices=["llama3_8b", "qwen25vl_7b"], default="llama3_8b")
    ap.add_argument("--reorder", action="store_true", help="information-flow chunk reordering (config 3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time the eager path only (no CUDA-graph replay)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sdpa-comparator", action="store_true", help="skip the torch-SDPA full-prefill comparator")
    ap.add_argument("--ncu", action="store_true", help="one warm step inside cudaProfilerStart/Stop, then exit")
    ap.add_argument("--simulate-ranks", type=int, default=1,
                    help="run the chunk-sharded path with R ranks as threads on one GPU (functional check)")
    return ap.parse_args()


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 20 ms during
    the timed region through NVML (nvidia-ml-py), falling back to
    `nvidia-smi -lms 200` when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksEventReason{HwSlowdown,HwThermalSlowdown,SwThermalSlowdown,SwPowerCap}

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.stop_evt = threading.Event()

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def begin(self):
        """Drop the samples taken before the timed region starts."""
        self.rows.clear()

    def _poll(self):
        nv, h = self.nvml
        while not self.stop_evt.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                bits = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.rows.append([mhz, self.max_mhz] + ["Active" if bits & b else "Not Active" for b in self.BITS])
            except Exception:
                pass
            self.stop_evt.wait(0.02)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.nvml is not None:
            self.stop_evt.set()
            self.thread.join()
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.proc.terminate()
            self.proc.wait()

        def num(x):
            try:
                return float(x)
            except (TypeError, ValueError):
                return None

        sm = [v for v in (num(r[0]) for r in self.rows) if v is not None]
        reasons = sorted({n for r in self.rows for n, v in zip(self.NAMES, r[2:]) if str(v).lower() == "active"})
        mx = next((v for v in (num(r[1]) for r in self.rows) if v is not None), None)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or os.environ.get("IFKV_FORCE_SHARDED"):
        import torch.distributed as dist

        # IFKV_FORCE_SHARDED=1 runs the chunk-sharded path even at world 1
        # (a one-rank NCCL communicator: every collective of the N-GPU bench
        # path on the one GPU this environment reaches).
        # IFKV_DIST_BACKEND=gloo runs the same TorchComm data path with every
        # rank on the visible GPUs round-robin (a functional check of the
        # multi-process path on a one-GPU box); the default is NCCL, one GPU per rank.
        backend = os.environ.get("IFKV_DIST_BACKEND", "nccl")
        if world > 1:  # communicator setup (ranks, channels, NVLS) visible in the driver's logs
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------


def model_config(args):
    import dataclasses

    import paper_2603_05353_b200 as P

    cfg = P.llama3_8b_config() if args.model == "llama3_8b" else P.qwen25vl_7b_config()
    if args.layers:
        cfg = dataclasses.replace(cfg, n_layers=args.layers)
    return cfg


def make_task(args, cfg):
    """C2/C3: fixed-size chunks; C4 (Qwen2.5-VL): 24 image-token chunks of
    1280 followed by 512-token text chunks up to the context length."""
    import paper_2603_05353_b200 as P

    if args.model == "qwen25vl_7b":
        lens = [1280] * 24
        while sum(lens) < args.ctx:
            lens.append(min(512, args.ctx - sum(lens)))
        cuts = tuple(np.cumsum(lens)[:-1].tolist())
        return P.SyntheticTask(kind="uniform_noise", total_length=sum(lens), fixed_size=None, boundaries=cuts,
                               prompt_length=32, vocab_size=cfg.vocab_size)
    return P.SyntheticTask(kind="uniform_noise", total_length=args.ctx, fixed_size=args.chunk, prompt_length=32,
                           vocab_size=cfg.vocab_size)


def workload_name(args, cfg, n_ctx, n_chunks, k):
    import paper_2603_05353_b200 as P

    base = "C2: Llama-3-8B shape" if args.model == "llama3_8b" else "C4: Qwen2.5-VL-7B LM shape"
    if args.reorder:
        base = base.replace("C2", "C3") + " + info-flow reorder"
    return (f"{base} ({cfg.n_layers}L, {cfg.n_heads}q/{cfg.kv_heads}kv heads, d_ff {cfg.d_ff}), {n_ctx} ctx in "
            f"{n_chunks} chunks, 32-token prompt, {args.ratio:.0%} recompute (k={k}), norm layer "
            f"{P.default_norm_layer(cfg.n_layers)}")


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def sdpa_full_prefill_ms(weights, toks, backend):
    """The ≤10 % comparator as SURVEY §8d defines it: a full bf16 causal prefill
    of the same context with torch + library attention (``backend``: a
    torch.nn.attention.SDPBackend), K/V written per layer; cuBLAS GEMMs.  Returns
    ms (CUDA events, second of two runs), or None when the backend refuses."""
    import torch
    import torch.nn.functional as F
    from torch.nn.attention import sdpa_kernel

    cfg = weights.config
    blk = weights.gu_block
    H, Hkv, Dh, d = cfg.n_heads, cfg.kv_heads, cfg.d_head, cfg.d_model
    n = int(toks.size)
    ids = torch.as_tensor(toks, device="cuda")
    pos = torch.arange(n, device="cuda", dtype=torch.float64)
    inv = cfg.rope_base ** (-torch.arange(0, Dh, 2, device="cuda", dtype=torch.float64) / Dh)
    ang = pos[:, None] * inv[None, :]
    cos, sin = ang.cos().float()[:, None, :], ang.sin().float()[:, None, :]

    def rope(x):  # [n, heads, Dh] interleaved pairs, fp32 math
        xf = x.float().view(n, x.shape[1], Dh // 2, 2)
        a, b = xf[..., 0], xf[..., 1]
        return torch.stack([a * cos - b * sin, a * sin + b * cos], dim=-1).view(n, x.shape[1], Dh).to(x.dtype)

    def rms(h, g):
        return (h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + 1e-6) * g).to(torch.bfloat16)

    def run():
        h = weights.embedding.index_select(0, ids).float()
        kv = []
        for lw in weights.layers:
            qkv = rms(h, lw.attn_norm) @ lw.wqkv.t()
            q, k, v = qkv.split([H * Dh, Hkv * Dh, Hkv * Dh], dim=-1)
            q, k = rope(q.view(n, H, Dh)), rope(k.view(n, Hkv, Dh))
            v = v.view(n, Hkv, Dh)
            kv.append((k, v))
            o = F.scaled_dot_product_attention(q.transpose(0, 1)[None], k.transpose(0, 1)[None],
                                               v.transpose(0, 1)[None], is_causal=True, enable_gqa=True)
            h = h + (o[0].transpose(0, 1).reshape(n, H * Dh) @ lw.wo.t()).float()
            gu = (rms(h, lw.mlp_norm) @ lw.wgu.t()).view(n, -1, 2, blk)  # gate/up interleaved in blk blocks
            g, u = gu[:, :, 0].reshape(n, cfg.d_ff), gu[:, :, 1].reshape(n, cfg.d_ff)
            h = h + ((F.silu(g.float()) * u.float()).to(torch.bfloat16) @ lw.wdown.t()).float()
        return kv

    try:
        with sdpa_kernel([backend]):
            times = []
            for _ in range(2):
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                out = run()
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
                del out
        return times[-1]
    except Exception:  # noqa: BLE001 -- backend not available for this shape/GPU
        return None


def run_ours(args, world, rank, local):
    import torch

    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200 import _native as N
    from paper_2603_05353_b200 import engine as E

    cfg = model_config(args)
    weights = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
    task = make_task(args, cfg)
    gen = P.generate_task(task, seed=rank)
    chunks, prompt = gen.chunks, gen.prompt_token_ids
    chunk_kvs = P.prefill_chunks(weights, chunks)  # prepared context in one store slab (not timed)
    sel_cfg = P.SelectionConfig(ratio=args.ratio)
    n_ctx = sum(c.local_length for c in chunks)
    torch.cuda.synchronize()

    def step(timer=None):
        return P.assemble_select_recompute(weights, chunk_kvs, chunks, prompt, sel_cfg, reorder=args.reorder,
                                           timer=timer)

    # the product path for repeated queries over one prepared context: the
    # whole query replayed as one CUDA graph (pipeline.QueryGraph), captured
    # during the warm-up; the eager path is timed beside it
    use_graph = not args.no_graph and not args.reorder and not args.ncu

    def gstep():
        return P.assemble_select_recompute(weights, chunk_kvs, chunks, prompt, sel_cfg, graph=True)

    for _ in range(args.warmup):
        res = step()
    del res
    torch.cuda.synchronize()
    if args.ncu:  # profiler capture range for ncu --profile-from-start off
        torch.cuda.profiler.start()
        res = step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return None

    # stage breakdown (untimed pass, stage events only), then kernel brackets
    # (another pass: their per-launch events would inflate the stage times)
    timer = P.StageTimer()
    res = step(timer)
    torch.cuda.synchronize()
    stages = timer.durations_ms()
    del res
    E.PROFILE = {}
    res = step()
    torch.cuda.synchronize()
    sel_h = res.selection.selected_numpy()
    margin = boundary_margin(res.selection.scores_numpy(), sel_h.size)
    prof = E.PROFILE
    E.PROFILE = None
    attn = prof.get("recompute_attn", [])
    attn_ms = [a.elapsed_time(b) for a, b, _ in attn]
    gem = [(a.elapsed_time(b), w) for a, b, w in prof.get("gemm", [])]
    pmm = [(a.elapsed_time(b), w) for a, b, w in prof.get("prompt_mm", [])]
    del res
    # the same selection in the float64 scoring mode (exact.py, untimed): how
    # many near-tied pairs the fp32-accurate fast path orders differently from
    # a float64 scorer at this instance (the reference scores in float64)
    sel_parity = None
    if not args.reorder and world == 1:
        t64 = time.perf_counter()
        r64 = P.assemble_select_recompute(weights, chunk_kvs, chunks, prompt,
                                          P.SelectionConfig(ratio=args.ratio, score_precision="fp64"))
        torch.cuda.synchronize()
        s64 = r64.selection.selected_numpy()
        sel_parity = {"k": int(sel_h.size), "swapped_pairs_vs_fp64_scoring": int(np.setxor1d(sel_h, s64).size // 2),
                      "fp64_query_ms": (time.perf_counter() - t64) * 1e3,
                      "note": "score_precision='fp64' reproduces the float64 reference's set at any margin "
                              "(tests/test_gpu_headline.py); the timed path scores fp32-accurately"}
        del r64

    if use_graph:  # capture (first call) + warm replays, after the eager stage / kernel-bracket passes
        for _ in range(args.warmup):
            res = gstep()
        del res
        torch.cuda.synchronize()

    # timed region
    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)  # (nvidia-smi fallback: let the sampler start)
    torch.cuda.synchronize()
    launches0 = N.LAUNCH_COUNT[0]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.begin()  # samples count from here (the timed region) on
    ev0.record()
    for _ in range(args.steps):
        res = gstep() if use_graph else step()
        del res
    ev1.record()
    torch.cuda.synchronize()
    launches = N.LAUNCH_COUNT[0] - launches0
    if use_graph:  # entry-point calls recorded in the graph, once per replay
        from paper_2603_05353_b200.pipeline import query_graph

        launches = query_graph(weights, chunk_kvs, chunks, len(prompt), sel_cfg).launches * args.steps
    clk = clocks.stop()
    barrier(world)
    ms = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms, world)
    value = n_ctx * world / (ms / 1e3)
    # e2e through the public API with host buffers in and out, right after the
    # device-timed loop (same thermal state; the eager comparison runs after)
    e2e = None
    if not args.no_e2e:
        times = []
        h2d = d2h = 0
        for _ in range(max(2, min(args.steps, 5))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = P.assemble_select_recompute(weights, chunk_kvs, chunks, np.array(prompt), sel_cfg,
                                              reorder=args.reorder, graph=use_graph)
            sel_host = res.selection.selected_numpy()
            sc_host = res.selection.scores_numpy()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            h2d = prompt.nbytes + (0 if use_graph else res.cache.token_ids.nbytes)  # graph: token ids are static
            d2h = sel_host.size * 8 + sc_host.size * 4
            del res
        e2e_ms = max_over_ranks(statistics.median(times) * 1e3, world)
        e2e = {"value": n_ctx * world / (e2e_ms / 1e3), "unit": "ctx tok/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    eager_ms = None
    if use_graph:  # the same steps through the eager path (one launch per kernel from Python)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            res = step()
            del res
        ev1.record()
        torch.cuda.synchronize()
        eager_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)

    # roofline of the dominant kernel of ours: recompute attention (tensor-bound)
    H, Dh, L = cfg.n_heads, cfg.d_head, cfg.n_layers
    flops_per_launch = 4.0 * H * Dh * float(np.sum(sel_h + 1))  # (selected in the final, permuted layout)
    attn_avg_ms = float(np.mean(attn_ms)) if attn_ms else None
    achieved = flops_per_launch / (attn_avg_ms / 1e3) / 1e12 if attn_avg_ms else None
    peak = PEAKS["bf16_tflops_sustained"]
    roof = {"kernel": "ifkv recompute_attn (tcgen05)", "bound": "tensor", "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s", "frac": achieved / peak if achieved else None,
            "traffic": ncu_traffic("recompute_attn_tc"), "traffic_source": f"ncu --set full, {TRAFFIC_FILE.name}",
            "peak_source": PEAKS["source"] + " sustained bf16",
            "algorithmic_flops_per_launch": flops_per_launch, "avg_launch_ms": attn_avg_ms,
            "launches_per_step": len(attn_ms), "share_of_step": float(np.sum(attn_ms)) / ms if attn_ms else None}
    # Kernel 1 (rotate_heads to global positions) runs inside the assemble
    # gather (one read of every chunk row, one write of the decode-layout slab)
    asm = [(a.elapsed_time(b), w) for a, b, w in prof.get("assemble_rotate", [])]
    rot_roof = None
    if asm:
        t_a, b_a = sum(t for t, _ in asm) / len(asm), sum(w for _, w in asm) / len(asm)
        ach = b_a / (t_a / 1e3) / 1e9
        rot_roof = {"kernel": "ifkv assemble_gather_rotate (assemble + Kernel 1 fused)", "bound": "hbm",
                    "achieved": ach, "peak": PEAKS["hbm_gbs"], "unit": "GB/s", "frac": ach / PEAKS["hbm_gbs"],
                    "frac_of_8tbs_spec": ach / HBM_SPEC_GBS, "avg_launch_ms": t_a,
                    "algorithmic_bytes_per_launch": b_a, "launches_per_step": len(asm),
                    "traffic": ncu_traffic("assemble_gather")}
    sct_roof = {"note": "the RoPE + in-place K/V scatter runs in the QKV GEMM epilogue (roofline_gemm)"}

    gemm_roof = None
    if gem:  # the tcgen05 projection GEMMs of the recompute (fused epilogues), all launches of one step
        t_g, f_g = sum(t for t, _ in gem), sum(w for _, w in gem)
        ach = f_g / (t_g / 1e3) / 1e12
        gemm_roof = {"kernel": "ifkv gemm_pair (tcgen05 cta_group::2, fused epilogues)", "bound": "tensor",
                     "achieved": ach, "peak": PEAKS["bf16_tflops_sustained"], "unit": "TFLOP/s",
                     "frac": ach / PEAKS["bf16_tflops_sustained"], "launches_per_step": len(gem),
                     "ms_per_step": t_g, "algorithmic_flops_per_step": f_g,
                     "peak_source": PEAKS["source"] + " sustained bf16 (cuBLAS)"}

    pmm_roof = None
    if pmm:
        # scoring-pass weight-stream GEMMs, timed back to back (inside the step
        # their event brackets would also count the host-paced gaps of the
        # selection): every projection of the scoring layers once, weights
        # streamed from HBM (each layer's 436 MB exceeds L2), fixed split3 input
        nl = P.default_norm_layer(cfg.n_layers)
        mats = [w for lw in weights.layers[: nl + 1] for w in (lw.wqkv, lw.wo, lw.wgu, lw.wdown)]
        xs = {m.shape[1]: torch.randn((3, 32, m.shape[1]), device="cuda").to(torch.bfloat16) for m in mats}
        for m in mats[:4]:  # weights are stored [N][K]
            E.mm_parts(xs[m.shape[1]], m)
        torch.cuda.synchronize()
        pa, pb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pa.record()
        for m in mats:
            E.mm_parts(xs[m.shape[1]], m)
        pb.record()
        torch.cuda.synchronize()
        t_p = pa.elapsed_time(pb)
        b_p = float(sum(m.numel() * 2 + 3 * 32 * m.shape[1] * 2 + E.prompt_mm_splits(m.shape[0], m.shape[1], 32,
                                                                                         E._sm_count()) * 32 * m.shape[0] * 4
                        for m in mats))
        ach = b_p / (t_p / 1e3) / 1e9
        pmm_roof = {"kernel": "ifkv prompt_mm (tcgen05 weight stream)", "bound": "hbm", "achieved": ach,
                    "peak": PEAKS["hbm_gbs"], "unit": "GB/s", "frac": ach / PEAKS["hbm_gbs"],
                    "frac_of_8tbs_spec": ach / HBM_SPEC_GBS, "ms_all_layers": t_p,
                    "algorithmic_bytes": b_p, "launches": len(mats),
                    "how": f"the {len(mats)} projections of layers 0..{nl} back to back, CUDA events",
                    "traffic": ncu_traffic("prompt_mm"),
                    "traffic_note": "ncu DRAM bytes of one launch (layer-0 gate|up, 235 MB of weights)"}

    # comparator: full bf16 prefill of the same context through the same kernels
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    toks = np.concatenate([c.token_ids for c in chunks])
    ours_ms = []
    for _ in range(2):  # the first run also allocates the 32K-row activations
        torch.cuda.synchronize()
        ea.record()
        full = P.full_prefill(weights, toks)
        eb.record()
        torch.cuda.synchronize()
        ours_ms.append(ea.elapsed_time(eb))
        del full
    full_by = {"ours (same kernels)": ours_ms[-1]}
    if not args.no_sdpa_comparator and n_ctx <= 65536:  # (at 128K the torch prefills alone take minutes)
        from torch.nn.attention import SDPBackend

        for name, be in (("torch SDPA cuDNN", SDPBackend.CUDNN_ATTENTION), ("torch SDPA flash", SDPBackend.FLASH_ATTENTION)):
            t = sdpa_full_prefill_ms(weights, toks, be)
            if t is not None:
                full_by[name] = t
        torch.cuda.empty_cache()
    full_ms = min(full_by.values())  # best of: the comparator is the fastest full prefill measured

    # the path's input producer: all chunks prefilled in one
    # block-diagonal layer stack, against the same-kernel full prefill's MFU
    cp = None
    if n_ctx <= 65536:
        torch.cuda.synchronize()
        cp_ms = []
        for _ in range(2):
            ea.record()
            kv_b = P.prefill_chunks(weights, chunks)
            eb.record()
            torch.cuda.synchronize()
            cp_ms.append(ea.elapsed_time(eb))
            del kv_b
        lens = np.array([c.local_length for c in chunks], dtype=np.float64)
        lin = lambda n: 2.0 * n * ((cfg.n_layers - 1) * cfg.params_per_layer() + cfg.d_model * 2 * cfg.kv_dim)  # noqa: E731
        attn = lambda tri: 4.0 * cfg.n_heads * cfg.d_head * (cfg.n_layers - 1) * tri  # noqa: E731
        f_chunks = lin(n_ctx) + attn(float(np.sum(lens * (lens + 1) / 2)))
        f_full = lin(n_ctx) + attn(n_ctx * (n_ctx + 1) / 2.0)
        peak = PEAKS["bf16_tflops_sustained"] * 1e12
        cp = {"ms": cp_ms[-1], "chunks": len(chunks), "tflops": f_chunks / 1e12,
              "mfu_of_sustained": f_chunks / (cp_ms[-1] / 1e3) / peak,
              "full_prefill_mfu_of_sustained": f_full / (full_by["ours (same kernels)"] / 1e3) / peak,
              "how": "P.prefill_chunks: one block-diagonal causal layer stack over all chunks into one store slab"}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "ctx tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (reference generate_task uniform_noise tokens; random-init weights, GPU-drawn N(0,1)/sqrt(fan_in))",
        "config": {"workload": workload_name(args, cfg, n_ctx, len(chunks), sel_h.size),
                   "ctx_tokens": n_ctx, "chunks": len(chunks), "recompute_ratio": args.ratio,
                   "selected": int(sel_h.size), "parallelism": f"replicas x{world}",
                   "l2": "inputs larger than L2 (4.3 GB KV slab + 16 GB weights per step)",
                   "execution": ("CUDA-graph replay of the whole query (pipeline.QueryGraph, captured in the warm-up)"
                                 if use_graph else "eager (one launch per kernel from Python)")},
        "eager_ms_per_step": eager_ms,
        "stages_ms": stages,
        "full_prefill_ms": full_ms,
        "full_prefill_ms_by": full_by,
        "chunk_prefill": cp,
        "ratio_vs_full_prefill": ms / full_ms,
        "boundary_margin": margin,
        "selection_parity": sel_parity,
        "roofline": roof,
        "roofline_kernel1": rot_roof,
        "roofline_scatter": sct_roof,
        "roofline_gemm": gemm_roof,
        "roofline_prompt_mm": pmm_roof,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    return line


# ---------------------------------------------------------------------------
# N GPUs: one context chunk-sharded across ranks, strong scaling
# ---------------------------------------------------------------------------


def run_sharded(args, comm, world, rank, sync):
    """Every rank holds the chunks it owns (zig-zag), scores them, merges the
    per-layer softmax states and the top-k candidates with the other ranks,
    and recomputes its own selected tokens with attention over all ranks'
    keys.  value = context tokens / step time (max over ranks)."""
    import torch

    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200 import sharding as SH

    cfg = model_config(args)
    weights = P.DeviceWeights.random(cfg, seed=7, precision="bf16")
    task = make_task(args, cfg)
    gen = P.generate_task(task, seed=0)
    chunks, prompt = gen.chunks, gen.prompt_token_ids
    shard = SH.make_shard([c.local_length for c in chunks], rank, world)
    my_kvs = [P.prefill_chunk(weights, chunks[c]) for c in shard.chunk_ids]
    sel_cfg = P.SelectionConfig(ratio=args.ratio)
    n_ctx = sum(c.local_length for c in chunks)

    budget = sel_cfg.resolve_budget(n_ctx)

    def step(prompt_ids):
        if args.reorder:  # first pass per rank, permutation from the all-gathered importances
            _, _, pshard, local = SH.sharded_reorder(weights, chunks, my_kvs, shard, prompt_ids, budget, comm)
        else:
            pshard, local = shard, P.assemble(my_kvs)
        res = SH.sharded_select(weights, pshard, local, prompt_ids, sel_cfg, comm)
        SH.sharded_recompute(weights, pshard, local, res.selected, comm)
        return res

    from paper_2603_05353_b200 import _native as N

    for _ in range(args.warmup):
        res = step(prompt)
    torch.cuda.synchronize()
    sync()
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    launches0 = N.LAUNCH_COUNT[0]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.begin()
    ev0.record()
    for _ in range(args.steps):
        res = step(prompt)
    ev1.record()
    torch.cuda.synchronize()
    launches = N.LAUNCH_COUNT[0] - launches0
    clk = clocks.stop()
    sync()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_all = comm.all_gather(torch.tensor([ms], dtype=torch.float64, device="cuda"))
    ms = max(float(x.item()) for x in ms_all)
    # e2e: host prompt ids in, selected indices out, through the sharded API
    times = []
    for _ in range(max(2, min(args.steps, 3))):
        torch.cuda.synchronize()
        sync()
        t0 = time.perf_counter()
        res = step(np.array(prompt))
        sel_host = res.selected.cpu().numpy()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    e2e_all = comm.all_gather(torch.tensor([statistics.median(times) * 1e3], dtype=torch.float64, device="cuda"))
    e2e_ms = max(float(x.item()) for x in e2e_all)
    return {
        "metric": METRIC,
        "value": n_ctx / (ms / 1e3),
        "unit": "ctx tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (reference generate_task uniform_noise tokens; random-init weights)",
        "config": {"workload": f"{'C3' if args.reorder else 'C2'} chunk-sharded over {world} ranks (zig-zag chunk "
                               f"ownership, {'per-rank reorder first pass + importance all-gather, ' if args.reorder else ''}"
                               f"NCCL softmax-state merges + top-k candidate all-gather + sparse-query partial "
                               f"attention all-to-all)",
                   "ctx_tokens": n_ctx, "chunks": len(chunks), "recompute_ratio": args.ratio,
                   "selected": int(sel_host.size), "parallelism": f"chunk-sharded x{world}",
                   "l2": "inputs larger than L2"},
        "e2e": {"value": n_ctx / (e2e_ms / 1e3), "unit": "ctx tok/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(prompt.nbytes), "d2h_bytes_per_step": int(sel_host.size * 8)},
        "roofline": None,
        "gpu_launches": int(launches),
        "clocks": clk,
    }


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (NumPy port of the reference) on a bounded sample
# ---------------------------------------------------------------------------


def cpu_sample_setup(args, seed=0):
    """Inputs of the CPU sample: a 2-layer model at Llama-3-8B width (f32),
    the full context's chunk KVs for those 2 layers, a prompt."""
    import oracle as O

    try:
        from threadpoolctl import threadpool_info

        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    d, h, hkv, dh, dff, vocab = 4096, 32, 8, 128, 14336, 4096
    n, m, chunk = args.ctx, 32, args.chunk
    k = int(np.ceil(args.ratio * n))

    class Cfg:
        n_layers, n_heads, n_kv_heads, d_head, d_model, d_ff, vocab_size = 2, h, hkv, dh, d, dff, vocab
        rope_base, max_position = 500000.0, 1 << 20

    class Layer:
        pass

    def mat(r, c, s):
        return (rng.standard_normal((r, c), dtype=np.float32) * np.float32(s))

    layers = []
    for _ in range(2):
        lw = Layer()
        lw.attn_norm = np.ones(d, np.float32)
        lw.mlp_norm = np.ones(d, np.float32)
        lw.wq, lw.wk, lw.wv, lw.wo = mat(d, d, d ** -0.5), mat(d, hkv * dh, d ** -0.5), mat(d, hkv * dh, d ** -0.5), \
            mat(d, d, d ** -0.5)
        lw.w_gate, lw.w_up, lw.w_down = mat(d, dff, d ** -0.5), mat(d, dff, d ** -0.5), mat(dff, d, dff ** -0.5)
        layers.append(lw)

    class W:
        pass

    w = W()
    w.config, w.layers = Cfg, layers
    w.embedding = mat(vocab, d, 1.0)
    w.final_norm, w.out_head = np.ones(d, np.float32), mat(d, 8, 1.0)
    chunks = []
    for c in range(n // chunk):
        kk = rng.standard_normal((2, chunk, hkv, dh), dtype=np.float32)
        vv = rng.standard_normal((2, chunk, hkv, dh), dtype=np.float32)
        chunks.append(O.Chunk(f"c{c}", rng.integers(0, vocab, chunk), kk, vv, np.arange(chunk), 0))
    prompt = rng.integers(0, vocab, m)
    sel = np.sort(rng.choice(n, k, replace=False))[::8]  # 1/8 of the selected rows (cost is linear in rows)
    return dict(w=w, chunks=chunks, prompt=prompt, sel=sel, threads=threads, n=n, m=m, chunk=chunk, k=k)


def cpu_sample(args, inp):
    """One scoring pass (layer 0 full + layer 1 captured) and one recompute
    pass (layer 0 full + layer 1 K/V) at Llama-3-8B width on the full context
    (oracle, f32, all host threads), extrapolated to the 32-layer path with
    norm layer 19: t = asm + (19 + 0.3)/1.3 x score2 + (31 + 0.1)/1.1 x rec2.
    Returns (extrapolated seconds, sample description, threads)."""
    import oracle as O

    w, chunks, prompt, sel = inp["w"], inp["chunks"], inp["prompt"], inp["sel"]
    threads, n, m, chunk, k = inp["threads"], inp["n"], inp["m"], inp["chunk"], inp["k"]
    t0 = time.perf_counter()
    cache = O.assemble(chunks)
    t_asm = time.perf_counter() - t0
    ctx, prm = O.assign_positions("GLOBAL", [chunk] * (n // chunk), m)
    t0 = time.perf_counter()
    O.score_attention_norm(w, cache, prompt, np.concatenate(ctx), prm, norm_layer=1)
    t_score2 = time.perf_counter() - t0  # layer 0 full + layer 1 capture ~ 1.3 layers
    t0 = time.perf_counter()
    O.recompute_selected(w, cache, sel)
    t_rec2 = 8.0 * (time.perf_counter() - t0)  # 1/8 of the rows; layer 0 full + layer 1 K/V only
    t_total = t_asm + (19 + 0.3) / 1.3 * t_score2 + (31 + 0.1) / 1.1 * t_rec2
    desc = (f"oracle f32 on {threads} threads: Llama-3-8B width, 2 layers, {n} ctx, k={k}; measured assemble "
            f"{t_asm:.2f}s, 2-layer scoring {t_score2:.2f}s, 2-layer recompute of k/8 rows x 8 = {t_rec2:.2f}s; "
            f"extrapolated to "
            f"32 layers / norm layer 19 as asm + 14.8 x score2 + 28.3 x rec2")
    return t_total, desc, threads


REF_DIR = ROOT / "baseline" / "_ref"  # the reference package installed (pip --target), git-ignored


def reference_c1_calibration(reps: int = 5):
    """The REAL reference (chunkkv from baseline/_ref) on BASELINE config 1,
    assemble + run_selection + make_plan + recompute_selected through its own
    public API (harness.py:449-456), beside the oracle port on the same
    inputs, in f32 and f64, on this host's cores: how fast the port used for
    the C2 extrapolation is relative to the reference itself."""
    import oracle as O

    if not (REF_DIR / "chunkkv").exists():
        return {"unavailable": f"{REF_DIR} not installed (pip install --target baseline/_ref)"}
    sys.path.insert(0, str(REF_DIR))
    try:
        import chunkkv as ck
    finally:
        sys.path.remove(str(REF_DIR))
    out = {"config": "C1: 2 layers, 4 heads x 128, d_ff 1792, 8 x 256 ctx + 32 prompt, r = 0.15 (k = 308)",
           "reps": reps, "threads": _blas_threads()}
    for prec in ("f32", "f64"):
        cfg = ck.ModelConfig(n_layers=2, n_heads=4, d_model=512, d_head=128, d_ff=1792, vocab_size=1024,
                             max_position=8192)
        w = ck.init_weights(cfg, 7, precision=prec)
        task = ck.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32,
                                vocab_size=1024)
        g = ck.generate_task(task, 0)
        kvs = [ck.prefill_chunk(w, c) for c in g.chunks]
        sel_cfg = ck.SelectionConfig(ratio=0.15)

        def ref_step():
            cache = ck.assemble(kvs)
            res = ck.run_selection(w, g.chunks, cache, g.prompt_token_ids, sel_cfg)
            ck.recompute_selected(w, cache, ck.make_plan(cache, res.selected))
            return res.selected

        ochunks = [O.Chunk(c.chunk_id, np.asarray(c.token_ids), np.stack(c.keys), np.stack(c.values),
                           np.asarray(c.prefill_positions), 0) for c in kvs]

        def port_step():
            cache = O.assemble(ochunks)
            _, sel = O.run_selection(w, cache, g.prompt_token_ids, ratio=0.15)
            O.recompute_selected(w, cache, *O.make_plan(cache.context_length, sel))
            return sel

        tr, tp = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            sel_r = ref_step()
            tr.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            sel_p = port_step()
            tp.append(time.perf_counter() - t0)
        r_ms, p_ms = statistics.median(tr) * 1e3, statistics.median(tp) * 1e3
        out[prec] = {"reference_ms": r_ms, "port_ms": p_ms, "port_over_reference_time": p_ms / r_ms,
                     "same_selected_set": bool(np.array_equal(np.sort(np.asarray(sel_r)), sel_p))}
    return out


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, world, rank):
    if rank != 0:
        return None
    times = []
    desc, threads = "", 1
    inp = cpu_sample_setup(args)
    for i in range(args.warmup + args.steps):
        t, desc, threads = cpu_sample(args, inp)
        if i >= args.warmup:
            times.append(t)
    t = statistics.median(times)
    value = args.ctx / t
    return {"metric": METRIC, "value": value, "unit": "ctx tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "extrapolated": True,
            "extrapolation": "each step times a 2-layer Llama-width sample of the C2 workload on the host cores "
                             "(~10-30 s) and extrapolates it to 32 layers / norm layer 19; ms_per_step is that "
                             "extrapolated full-workload time, not the wall time of the step",
            "config": {"workload": "C2 sample (see cpu_baseline.sample)", "ctx_tokens": args.ctx},
            "cpu_baseline": {"value": value, "unit": "ctx tok/s", "cores": threads, "kind": "port", "sample": desc},
            "reference_c1_calibration": reference_c1_calibration(),
            "e2e": {"value": value, "unit": "ctx tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if os.environ.get("IFKV_BENCH_WATCHDOG"):  # debugging: dump every thread's stack and exit after N s
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["IFKV_BENCH_WATCHDOG"]), exit=True)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        line = run_reference(args, world, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    world, rank, local = dist_setup()
    if world > 1 or os.environ.get("IFKV_FORCE_SHARDED"):
        from paper_2603_05353_b200.sharding import TorchComm

        import torch.distributed as dist

        line = run_sharded(args, TorchComm(), world, rank, dist.barrier)
        clk = None
        if rank == 0:
            print(json.dumps(line), flush=True)
        dist.destroy_process_group()
        return
    if args.simulate_ranks > 1:
        from paper_2603_05353_b200.sharding import ThreadComm

        import torch

        def body(comm):
            return run_sharded(args, comm, comm.world, comm.rank,
                               lambda: comm.all_gather(torch.zeros(1, device="cuda")))

        line = ThreadComm.run(args.simulate_ranks, body)[0]
        line["n_gpus"] = 1
        line["simulated_ranks"] = args.simulate_ranks
        line["scaling"] = "none (ranks simulated as threads on one GPU: functional check, not a scaling number)"
        print(json.dumps(line), flush=True)
        return
    line = run_ours(args, world, rank, local)
    if line is None:
        return
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t, desc, threads = cpu_sample(args, cpu_sample_setup(args))
        line["cpu_baseline"] = {"value": args.ctx / t, "unit": "ctx tok/s", "cores": threads, "kind": "port",
                                "sample": desc, "extrapolated": True,
                                "reference_c1_calibration": reference_c1_calibration()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
