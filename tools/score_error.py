"""Where does the scoring error come from?  Llama-3-8B width, 4 layers, 32K
context: GPU attention-norm scores (several arithmetic variants) against the
float64 oracle on identical inputs.  python tools/score_error.py"""
import dataclasses, sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import oracle as O  # noqa: E402
import paper_2603_05353_b200 as P  # noqa: E402
from paper_2603_05353_b200.model import DeviceLayer  # noqa: E402
from paper_2603_05353_b200 import engine as E  # noqa: E402
from helpers import oracle_chunk  # noqa: E402
from test_gpu_headline import oracle_weights  # noqa: E402

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
cfg = dataclasses.replace(P.llama3_8b_config(), n_layers=4)
dw = P.DeviceWeights.random(cfg, seed=7)
task = P.SyntheticTask(kind="uniform_noise", total_length=ctx, fixed_size=2048, prompt_length=32, vocab_size=cfg.vocab_size)
g = P.generate_task(task, 0)
kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
cache = P.assemble(kvs)
nl = 2
t0 = time.time()
ow = oracle_weights(dw, nl + 1)
oc = O.assemble([oracle_chunk(c) for c in kvs])
ref, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
print(f"oracle {time.time() - t0:.1f}s", flush=True)
s = np.sort(ref)[::-1]
k = sel.size
print(f"gap_k rel {(s[k-1] - s[k]) / s[k-1]:.2e}")


def report(name, got):
    got = np.asarray(got, np.float64)
    rel = np.abs(got - ref) / ref
    same = np.array_equal(np.sort(np.argsort(-got, kind="stable")[:k]), sel)
    print(f"{name:40s} max rel {rel.max():.2e} median {np.median(rel):.2e} set-equal {same}", flush=True)


def run(impl="auto", w=dw, c=cache):
    res = P.run_selection(w, g.chunks, c, g.prompt_token_ids, P.SelectionConfig(ratio=0.15))
    return res.scores_numpy()


report("bf16 default (tcgen05)", run())
# SIMT attention kernels (GEMMs still tensor-core)
orig = E.prompt_forward
E.prompt_forward = lambda *a, **kw: orig(*a, **{**kw, "impl": "simt"})
report("bf16, SIMT attention", run())
E.prompt_forward = orig
# tensor-core GEMMs on our pair GEMM instead of prompt_mm
E.PROMPT_MM = False
report("bf16, pair GEMM instead of prompt_mm", run())
E.PROMPT_MM = True
# fp32 mode: fp32 weights/KV, IEEE torch.mm (TF32 off), SIMT kernels
torch.backends.cuda.matmul.allow_tf32 = False
w32 = P.DeviceWeights(cfg, "f32", dw.embedding.float(), [DeviceLayer(l.attn_norm, l.wqkv.float(), l.wo.float(), l.mlp_norm,
                      l.wgu.float(), l.wdown.float()) for l in dw.layers], dw.final_norm, dw.out_head.float())
c32 = P.assemble([dataclasses.replace(x, keys=x.keys.float(), values=x.values.float()) for x in kvs])
report("fp32 mode (IEEE)", run(w=w32, c=c32))
