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


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle.oracle as O
    lpt_partition, shard_rows = _lpt()
    b = make_batch(name, 0)
    # replicated trajectory metadata -> identical advantages on every rank
    adv, inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P)
    mine = lpt_partition(b.lengths, world)[rank]
    rows, cu_l = shard_rows(b.cu_seqlens, mine)
    bits = b.logits_bits(rows)
    # rank-local packing; trajectory j of this rank reads adv[mine[j]] (the traj_index map)
    rr = O.rows(np.arange(len(rows)), bits, b.V, b.target_ids[rows], b.logp_behav[rows], cu_l,
                adv[mine], inv[mine], 0.2, want_dlogits=False)
    J_local, _ = O.objective_tokens(cu_l, inv[mine], rr.term)
    stats = torch.tensor([J_local, float(len(rows)), float(rr.clipped.sum())], dtype=torch.float64)
    dist.all_reduce(stats)
    if rank == 0:
        out.put(stats.numpy().tolist())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["ragged", "mid32k"])
def test_gloo_world2_sharded_objective(name):
    import oracle.oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    b = make_batch(name, 0)
    ref = O.run_batch(b, b.logits_bits(), want_dlogits=False)
    assert got[1] == b.T
    assert got[2] == ref["n_clipped"]
    assert abs(got[0] - ref["J"]) <= 1e-12 * max(1.0, abs(ref["J"]))
