"""-m gpu: the data-parallel step of bench.py at world 2 and 4 with the ranks emulated one
after another on one GPU: LPT token-balanced trajectory shards, each rank with
its own token arrays only (grpo_async_validate_local: trajectory checks over all N, token
checks over its trajectories), its fused-loss chunks accumulating into its packed fp64
partials [stats, token-level validation counts], then the exchange -- every rank's vector
gathered in rank order and summed by grpo_async_combine_ranks -- and
grpo_async_validate_combine.  Checked: the combined summary equals the unsharded
validation field for field (faults injected on one rank's rows included), J equals the
oracle's under Z17, counters exact, and the combined vector is bit-identical run to run."""
import numpy as np
import pytest
import torch

import oracle.oracle as O
import paper_2604_26256_b200 as G
from synth.gen import make_batch
from tests.gpu_util import Z17_GUARD, near_boundary, to_dev_bits

pytestmark = pytest.mark.gpu


def _step(dev, b, bits, world, tgt_override=None):
    """One emulated multi-rank step; returns (combined vector, combined summary dict)."""
    tgt_all = b.target_ids if tgt_override is None else tgt_override
    loss = G.GrpoAsyncLoss()
    NP = G.NUM_STATS + 3
    gathered = torch.zeros((world, NP), dtype=torch.float64, device=dev)
    vos = []
    rep = dict(cu=torch.from_numpy(b.cu_seqlens).to(dev), gid=torch.from_numpy(b.group_ids).to(dev),
               ver=torch.from_numpy(b.version_ids).to(dev), rew=torch.from_numpy(b.rewards).to(dev))
    for rank, mine in enumerate(G.lpt_partition(b.lengths, world)):
        rows, cu_l = G.shard_rows(b.cu_seqlens, mine)
        t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to(dt).to(dev)
        sb = G.ShardedBatch(b.P, b.G, b.K, b.V, b.ld, b.tbs, b.v_theta, b.T, rep["cu"], rep["gid"],
                            rep["ver"], rep["rew"], t(cu_l, torch.int64), t(mine.astype(np.int32), torch.int32),
                            t(tgt_all[rows], torch.int64), t(b.logp_behav[rows], torch.float32),
                            None if b.token_version is None else t(b.token_version[rows], torch.int64))
        packed = gathered[rank]
        vo = loss.validate_local(sb, token_counts=packed[G.NUM_STATS:])
        adv, inv = loss.advantage(sb)
        ts = torch.zeros(len(mine), dtype=torch.float64, device=dev)
        lg = to_dev_bits(bits[rows], dev)
        half = len(rows) // 2   # two chunks per rank
        for b0, b1 in ((0, half), (half, len(rows))):
            loss.loss_chunk(lg[b0:b1], b0, b1 - b0, sb.target_ids[b0:b1], sb.logp_behav[b0:b1],
                            sb.local_cu, adv, inv, ts, packed[:G.NUM_STATS], traj_index=sb.traj_index,
                            V=b.V)
        vos.append(vo)
    glob = torch.empty(NP, dtype=torch.float64, device=dev)
    G.grpo_async_combine_ranks(gathered, world, NP, glob)
    for vo in vos:
        loss.validate_combine(vo, glob[G.NUM_STATS:])
    torch.cuda.synchronize()
    summaries = [vo.summary_dict() for vo in vos]
    assert all(sm == summaries[0] for sm in summaries)   # every rank holds the same verdict
    return glob.cpu().numpy(), summaries[0]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["ragged", "mid32k"])
def test_sharded_step_matches_oracle_and_is_deterministic(dev, name, world):
    b = make_batch(name, 5)
    bits = b.logits_bits()
    ref = O.run_batch(b, bits, want_dlogits=False)
    runs = [_step(dev, b, bits, world) for _ in range(3)]
    vec, summ = runs[0]
    for v, s in runs[1:]:
        assert np.array_equal(v, vec) and s == summ      # bit-identical, run to run
    assert summ == ref["validate"]["summary"]             # field for field, incl. C1 counts
    rr = ref["rows"]
    S_abs = float(np.sum(ref["inv_norm"][np.repeat(np.arange(b.N), b.lengths)] * np.abs(rr.term)))
    assert abs(vec[G.STAT_J] - ref["J"]) <= 1e-5 * max(abs(ref["J"]), Z17_GUARD * S_abs)
    assert vec[G.STAT_ROWS] == b.T
    flips = int(near_boundary(rr.r).sum())
    assert abs(vec[G.STAT_CLIPPED] - ref["n_clipped"]) <= flips
    assert vec[G.NUM_STATS:].tolist() == [float(ref["validate"]["summary"][k]) for k in
                                         ("n_c1_mixed", "n_bad_target", "n_bad_logp_behav")]


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_validation_fault_on_one_rank(dev, world):
    """A bad target on one row: only its owner sees it; the combined verdict is invalid on
    every rank, with the same counts as the unsharded validation."""
    b = make_batch("mid32k", 6)
    bits = b.logits_bits()
    tgt = b.target_ids.copy()
    tgt[int(b.cu_seqlens[3]) + 1] = b.V
    v = O.validate(b.version_ids, b.cu_seqlens, b.group_ids, tgt, P=b.P, V=b.V, G=b.G, tbs=b.tbs,
                   v_theta=b.v_theta, K=b.K, token_version=b.token_version, logp_behav=b.logp_behav)
    # the loss itself assumes validated input (targets in range): run it on the clean targets
    # and only the validation on the faulted ones
    loss = G.GrpoAsyncLoss()
    NP = G.NUM_STATS + 3
    gathered = torch.zeros((world, NP), dtype=torch.float64, device=dev)
    cu = torch.from_numpy(b.cu_seqlens).to(dev)
    vos = []
    for rank, mine in enumerate(G.lpt_partition(b.lengths, world)):
        rows, cu_l = G.shard_rows(b.cu_seqlens, mine)
        t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to(dt).to(dev)
        sb = G.ShardedBatch(b.P, b.G, b.K, b.V, b.ld, b.tbs, b.v_theta, b.T, cu,
                            t(b.group_ids, torch.int32), t(b.version_ids, torch.int64),
                            t(b.rewards, torch.float32), t(cu_l, torch.int64),
                            t(mine.astype(np.int32), torch.int32), t(tgt[rows], torch.int64),
                            t(b.logp_behav[rows], torch.float32), None)
        vos.append(loss.validate_local(sb, token_counts=gathered[rank, G.NUM_STATS:]))
    glob = torch.empty(NP, dtype=torch.float64, device=dev)
    G.grpo_async_combine_ranks(gathered, world, NP, glob)
    for vo in vos:
        loss.validate_combine(vo, glob[G.NUM_STATS:])
    torch.cuda.synchronize()
    for vo in vos:
        s = vo.summary_dict()
        assert s == v["summary"] and s["valid"] == 0 and s["n_bad_target"] == 1
