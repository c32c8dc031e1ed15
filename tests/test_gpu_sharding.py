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
