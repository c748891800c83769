"""Multi-GPU host logic on CPU (-m "not gpu"): the token-balanced LPT partition,
rank-local packing, and the one exchange step (all-reduce of the packed fp64
partials) with world_size 2 over gloo.  Per-shard partials come from the oracle
so the whole flow runs without a GPU; the CUDA per-shard path is covered by
tests/test_gpu_parity.py::test_sharded_equals_unsharded."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.gen import make_batch


def _lpt():
    # the partition lives in the product package's pure-Python plumbing; importing the
    # package needs libgrpo_async.so, which build() produces here without a GPU
    from paper_2604_26256_b200.api import lpt_partition, shard_rows
    return lpt_partition, shard_rows


@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["prod", "large", "dapo"])
def test_lpt_partition_is_token_balanced(name, R):
    lpt_partition, _ = _lpt()
    b = make_batch(name, 0)
    parts = lpt_partition(b.lengths, R)
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(b.N))            # trajectory-atomic, none dropped (C2)
    loads = np.array([b.lengths[p].sum() for p in parts])
    # LPT bound: max load <= mean + max single length
    assert loads.max() <= loads.mean() + b.lengths.max()
    if R > 1 and name != "large":
        assert loads.max() / loads.mean() < 1.01
    for p in parts:
        assert np.all(np.diff(p) > 0)


def test_shard_rows_packing():
    _, shard_rows = _lpt()
    b = make_batch("mid32k", 0)
    ids = np.array([3, 0, 7])
    rows, cu = shard_rows(b.cu_seqlens, ids)
    assert cu[-1] == len(rows) == b.lengths[ids].sum()
    for j, i in enumerate(ids):
        assert np.array_equal(rows[cu[j]:cu[j + 1]], np.arange(b.cu_seqlens[i], b.cu_seqlens[i + 1]))


def _rank_order_sum(gathered):
    """grpo_async_combine_ranks' definition (include/grpo_async.h): out[k] = g[0][k] + g[1][k]
    + ... in rank order -- restated here because the kernel needs a GPU."""
    acc = gathered[0].clone()
    for q in range(1, gathered.shape[0]):
        acc += gathered[q]
    return acc


def _worker(rank, world, port, name, out, fault):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle.oracle as O
    lpt_partition, shard_rows = _lpt()
    b = make_batch(name, 0)
    tgt_v = b.target_ids.copy()
    if fault is not None:  # a bad target on one row (token-level: counted by its owner only)
        tgt_v[fault] = b.V
    # replicated trajectory metadata -> identical advantages on every rank
    adv, inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P)
    mine = lpt_partition(b.lengths, world)[rank]
    rows, cu_l = shard_rows(b.cu_seqlens, mine)
    bits = b.logits_bits(rows)
    # rank-local packing; trajectory j of this rank reads adv[mine[j]] (the traj_index map)
    rr = O.rows(np.arange(len(rows)), bits, b.V, b.target_ids[rows], b.logp_behav[rows], cu_l,
                adv[mine], inv[mine], 0.2, want_dlogits=False)
    J_local, _ = O.objective_tokens(cu_l, inv[mine], rr.term)
    # token-level validation of this rank's trajectories only (its own token arrays)
    g_loc = np.zeros(len(mine), np.int32)  # group ids irrelevant to the token checks
    vloc = O.validate(b.version_ids[mine], cu_l, g_loc, tgt_v[rows], P=1, V=b.V,
                      G=len(mine), tbs=len(mine), v_theta=b.v_theta, K=b.K,
                      token_version=None if b.token_version is None else b.token_version[rows],
                      logp_behav=b.logp_behav[rows])["summary"]
    packed = torch.tensor([J_local, float(len(rows)), float(rr.clipped.sum()),
                           float(vloc["n_c1_mixed"]), float(vloc["n_bad_target"]),
                           float(vloc["n_bad_logp_behav"])], dtype=torch.float64)
    # the one exchange: all-gather in rank order, then the rank-order sum on every rank
    parts = [torch.zeros_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed)   # gloo has no all_gather_into_tensor
    gathered = torch.stack(parts)
    res = [_rank_order_sum(gathered) for _ in range(3)]
    assert all(torch.equal(res[0], r) for r in res[1:])           # run to run
    every = [torch.zeros_like(packed) for _ in range(world)]
    dist.all_gather(every, res[0])
    assert all(torch.equal(every[0], every[q]) for q in range(world))  # identical on every rank
    if rank == 0:
        out.put(res[0].numpy().tolist())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["ragged", "mid32k"])
def test_gloo_sharded_objective(name, world):
    """world 2 and 4 over gloo: LPT shards, rank-local oracle partials and token-level
    validation counts, all-gather + rank-order sum (bit-identical on every rank and run to
    run), equal to the unsharded oracle -- J to fp64 reordering, the counts exactly; a bad
    target injected on one rank's row reaches the combined count."""
    import oracle.oracle as O
    ctx = mp.get_context("spawn")
    b = make_batch(name, 0)
    for fault in (None, int(b.cu_seqlens[b.N // 2]) + 1):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, fault)) for r in range(world)]
        for p in procs:
            p.start()
        got = q.get(timeout=300)
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
        bb = make_batch(name, 0)
        if fault is not None:
            bb.target_ids[fault] = bb.V
        ref = O.run_batch(bb, bb.logits_bits(), want_dlogits=False) if fault is None else None
        v = O.validate(bb.version_ids, bb.cu_seqlens, bb.group_ids, bb.target_ids, P=bb.P, V=bb.V,
                       G=bb.G, tbs=bb.tbs, v_theta=bb.v_theta, K=bb.K, token_version=bb.token_version,
                       logp_behav=bb.logp_behav)["summary"]
        assert got[1] == bb.T
        assert (got[3], got[4], got[5]) == (v["n_c1_mixed"], v["n_bad_target"], v["n_bad_logp_behav"])
        if fault is None:
            assert got[2] == ref["n_clipped"]
            assert abs(got[0] - ref["J"]) <= 1e-12 * max(1.0, abs(ref["J"]))
        else:
            assert got[4] == 1
