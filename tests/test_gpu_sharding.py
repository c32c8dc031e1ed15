"""The chunk-sharded data path (zig-zag chunk ownership, per-layer softmax
state merges, candidate top-k merge, sparse-query partial attention with
all-to-all return) run end to end -- kernels included -- as R ranks on one
GPU (ThreadComm), against the oracle and the unsharded path."""

import numpy as np
import pytest

import oracle as O
from helpers import oracle_chunk, rel_err, to_np

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_select_and_recompute_match_oracle(cuda, world):
    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200 import sharding as SH

    cfg = P.c1_config()
    dw = P.DeviceWeights.from_host(P.init_weights(cfg, 7), "bf16")
    ow = dw.to_host()
    task = P.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32,
                           vocab_size=1024)
    g = P.generate_task(task, 1)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
    want = O.recompute_selected(ow, oc, *O.make_plan(oc.context_length, sel))
    wk, wv = O.decode_view(want, cfg.rope_base)

    def body(comm):
        shard = SH.make_shard([c.length for c in kvs], comm.rank, comm.world)
        local = P.assemble([kvs[i] for i in shard.chunk_ids])
        res = SH.sharded_select(dw, shard, local, g.prompt_token_ids, P.SelectionConfig(ratio=0.15), comm)
        SH.sharded_recompute(dw, shard, local, res.selected, comm)
        return shard, res.selected.cpu().numpy(), res.scores.double().cpu().numpy(), to_np(local.keys), \
            to_np(local.values), local.row_positions.copy()

    outs = SH.ThreadComm.run(world, body)
    full_scores = np.zeros(2048)
    gk, gv = np.zeros_like(wk[:, :2048]), np.zeros_like(wv[:, :2048])
    for shard, s_sel, s_scores, lk, lv, rp in outs:
        np.testing.assert_array_equal(s_sel, sel)  # every rank: the oracle's set, bit-exact
        full_scores[shard.global_rows] = s_scores
        gk[:, shard.global_rows] = lk
        gv[:, shard.global_rows] = lv
        np.testing.assert_array_equal(rp[: shard.global_rows.size], shard.global_rows)
    assert rel_err(full_scores, scores) <= 1e-4
    assert rel_err(gk, wk[:, :2048]) <= 1e-2
    assert rel_err(gv, wv[:, :2048]) <= 1e-2


def test_torchcomm_nccl_single_rank_path(cuda):
    """The TorchComm code path over a real NCCL communicator (world 1: every
    collective still runs through NCCL -- all_gather, variable-size gathers,
    list all_to_all with uneven and empty parts) end to end at C1, against
    the oracle.  Multi-GPU NCCL itself needs more than the one GPU here."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200 import sharding as SH

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = SH.TorchComm()
        a = torch.arange(12, dtype=torch.float32, device="cuda").view(6, 2)
        got = comm.all_to_all([a])
        assert torch.equal(got[0], a)
        e = comm.all_to_all([a[:0]])
        assert e[0].shape == (0, 2)
        gv = comm.all_gather_var(a[:5])
        assert torch.equal(gv[0], a[:5])

        cfg = P.c1_config()
        dw = P.DeviceWeights.from_host(P.init_weights(cfg, 7), "bf16")
        ow = dw.to_host()
        task = P.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32,
                               vocab_size=1024)
        g = P.generate_task(task, 2)
        kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
        oc = O.assemble([oracle_chunk(c) for c in kvs])
        scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
        want = O.recompute_selected(ow, oc, *O.make_plan(oc.context_length, sel))
        wk, wv = O.decode_view(want, cfg.rope_base)
        shard = SH.make_shard([c.length for c in kvs], 0, 1)
        local = P.assemble([kvs[i] for i in shard.chunk_ids])
        res = SH.sharded_select(dw, shard, local, g.prompt_token_ids, P.SelectionConfig(ratio=0.15), comm)
        SH.sharded_recompute(dw, shard, local, res.selected, comm)
        np.testing.assert_array_equal(res.selected.cpu().numpy(), sel)
        full = np.zeros(2048)
        full[shard.global_rows] = res.scores.double().cpu().numpy()
        assert rel_err(full, scores) <= 1e-4
        lk = np.zeros_like(wk[:, :2048])
        lk[:, shard.global_rows] = to_np(local.keys)
        assert rel_err(lk, wk[:, :2048]) <= 1e-2
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_reorder_matches_oracle(cuda, world):
    """Chunk-sharded information-flow reordering (first pass per rank, the
    importances all-gathered, one permutation everywhere, chunks kept on
    their ranks under the permuted global rows) then the sharded GLOBAL
    selection and recompute: permutation and selected set bit-exact against
    the oracle's reorder_and_reselect, recomputed K/V within the bf16 bar."""
    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200 import sharding as SH

    cfg = P.c1_config()
    dw = P.DeviceWeights.from_host(P.init_weights(cfg, 7), "bf16")
    ow = dw.to_host()
    task = P.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32,
                           vocab_size=1024)
    g = P.generate_task(task, 3)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    budget = 308
    perm, _, _, _, sel = O.reorder_and_reselect(ow, [oracle_chunk(c) for c in kvs], g.prompt_token_ids, budget)

    def body(comm):
        shard = SH.make_shard([c.length for c in kvs], comm.rank, comm.world)
        mine = [kvs[i] for i in shard.chunk_ids]
        p, _, pshard, local = SH.sharded_reorder(dw, g.chunks, mine, shard, g.prompt_token_ids, budget, comm)
        res = SH.sharded_select(dw, pshard, local, g.prompt_token_ids, P.SelectionConfig(topk=budget), comm)
        SH.sharded_recompute(dw, pshard, local, res.selected, comm)
        return p, res.selected.cpu().numpy(), pshard, to_np(local.keys)

    outs = SH.ThreadComm.run(world, body)
    for p, s, pshard, lk in outs:
        np.testing.assert_array_equal(p, perm)
        np.testing.assert_array_equal(s, sel)
    # the recomputed shards together equal the unsharded GPU reorder path's cache (decode layout)
    plan, cache, second = P.reorder_and_reselect(dw, g.chunks, g.prompt_token_ids, budget, prefilled=kvs)
    out = P.recompute_selected(dw, cache, P.make_plan(cache, second.selected))
    want = to_np(out.keys)
    got = np.zeros_like(want[:, :2048])
    for _, _, pshard, lk in outs:
        got[:, pshard.global_rows] = lk[:, : pshard.global_rows.size]
    assert rel_err(got, want[:, :2048]) <= 1e-2


# ---------------------------------------------------------------------------
# real processes: TorchComm over torch.distributed with world size 2
# ---------------------------------------------------------------------------


def _two_proc_rank(rank, world, store_path, backend, q):
    """One rank: the whole sharded path (select, recompute, reorder) at C1."""
    import torch
    import torch.distributed as dist

    import paper_2603_05353_b200 as P
    from paper_2603_05353_b200 import sharding as SH

    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    kw = {"device_id": torch.device("cuda", dev)} if backend == "nccl" else {}
    dist.init_process_group(backend, init_method=f"file://{store_path}", rank=rank, world_size=world, **kw)
    try:
        cfg = P.c1_config()
        dw = P.DeviceWeights.from_host(P.init_weights(cfg, 7), "bf16")
        task = P.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32,
                               vocab_size=1024)
        g = P.generate_task(task, 1)
        comm = SH.TorchComm()
        shard = SH.make_shard([c.local_length for c in g.chunks], rank, world)
        mine = [P.prefill_chunk(dw, g.chunks[i]) for i in shard.chunk_ids]
        local = P.assemble(mine)
        res = SH.sharded_select(dw, shard, local, g.prompt_token_ids, P.SelectionConfig(ratio=0.15), comm)
        SH.sharded_recompute(dw, shard, local, res.selected, comm)
        out = {"rows": shard.global_rows, "sel": res.selected.cpu().numpy(),
               "scores": res.scores.double().cpu().numpy(), "k": local.keys.double().cpu().numpy(),
               "v": local.values.double().cpu().numpy()}
        perm, imps, pshard, plocal = SH.sharded_reorder(dw, g.chunks, mine, shard, g.prompt_token_ids, 308, comm)
        res2 = SH.sharded_select(dw, pshard, plocal, g.prompt_token_ids, P.SelectionConfig(topk=308), comm)
        out.update(perm=perm, imps=imps, sel2=res2.selected.cpu().numpy())
        q.put((rank, out))
    except Exception as exc:  # surfaced in the parent
        import traceback

        q.put((rank, RuntimeError(traceback.format_exc())))
    finally:
        dist.destroy_process_group()


def test_two_process_torchcomm_path_matches_oracle(cuda):
    """Two OS processes, TorchComm over torch.distributed (NCCL when two GPUs
    are visible, else gloo with both ranks on the one GPU): sharded
    selection, recompute and reorder at C1, every rank's selected set and the
    reorder permutation bit-exact against the oracle, scores 1e-4, recomputed
    K/V 1e-2."""
    import os
    import tempfile

    import torch
    import torch.multiprocessing as mp

    import paper_2603_05353_b200 as P

    world = 2
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as tmp:
        procs = [ctx.Process(target=_two_proc_rank, args=(r, world, os.path.join(tmp, "store"), backend, q))
                 for r in range(world)]
        for p in procs:
            p.start()
        outs = dict(q.get(timeout=300) for _ in range(world))
        for p in procs:
            p.join(timeout=60)
    for v in outs.values():
        if isinstance(v, Exception):
            raise v
    cfg = P.c1_config()
    dw = P.DeviceWeights.from_host(P.init_weights(cfg, 7), "bf16")
    ow = dw.to_host()
    task = P.SyntheticTask(kind="uniform_noise", total_length=2048, fixed_size=256, prompt_length=32, vocab_size=1024)
    g = P.generate_task(task, 1)
    kvs = [P.prefill_chunk(dw, c) for c in g.chunks]
    oc = O.assemble([oracle_chunk(c) for c in kvs])
    scores, sel = O.run_selection(ow, oc, g.prompt_token_ids, ratio=0.15)
    want = O.recompute_selected(ow, oc, *O.make_plan(oc.context_length, sel))
    wk, wv = O.decode_view(want, cfg.rope_base)
    perm, imps, _, _, sel2 = O.reorder_and_reselect(ow, [oracle_chunk(c) for c in kvs], g.prompt_token_ids, 308)
    full = np.zeros(2048)
    gk, gv = np.zeros_like(wk[:, :2048]), np.zeros_like(wv[:, :2048])
    for r in range(world):
        o = outs[r]
        np.testing.assert_array_equal(o["sel"], sel)
        np.testing.assert_array_equal(o["perm"], perm)
        np.testing.assert_allclose(o["imps"], imps, rtol=1e-4)
        np.testing.assert_array_equal(o["sel2"], sel2)
        full[o["rows"]] = o["scores"]
        gk[:, o["rows"]] = o["k"][:, :o["rows"].size]
        gv[:, o["rows"]] = o["v"][:, :o["rows"].size]
    np.testing.assert_allclose(full, scores, rtol=1e-4, atol=0)
    assert rel_err(gk, wk[:, :2048]) <= 1e-2
    assert rel_err(gv, wv[:, :2048]) <= 1e-2
