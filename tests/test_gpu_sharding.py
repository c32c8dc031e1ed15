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
