"""-m gpu: the whole benchmark step (bench.py's workload `prod`, seed 0, 131072-row
resident chunk, default plan) and the other BASELINE.json configurations at full size --
`dapo` (32 x 16, lengths to 20k), `stale` (K = 8, partial-rollout C1_MIXED trajectories)
and `large` (V = 262144, rows split over two-SM clusters) -- against full-batch golden
values written by scripts/make_golden_full.py from the fp64 oracle alone (every row of
the batch through oracle_rows)."""
import json
import os

import numpy as np
import pytest
import torch

import paper_2604_26256_b200 as G
import synth.gpu as SG
from synth.gen import make_batch

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name,seed,R", [("prod", 0, 131072), ("dapo", 0, 131072), ("stale", 0, 65536),
                                         ("large", 0, 65536)])
def test_full_batch_against_oracle_golden(dev, name, seed, R):
    path = os.path.join(GOLD, f"{name}_seed{seed}_R{R}.json")
    gold = json.load(open(path))
    b = make_batch(name, seed, period=R)
    assert b.T == gold["T"] and b.N == gold["N"]
    lg = torch.empty((R, b.ld), dtype=torch.int16, device=dev)
    dl = torch.empty_like(lg)
    SG.fill_logits(lg, b.logits, 0, R, b.V)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    vo = loss.validate(db)
    adv, inv = loss.advantage(db)
    traj_sum = torch.zeros(b.N, dtype=torch.float64, device=dev)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    for c0 in range(0, b.T, R):
        n = min(R, b.T - c0)
        loss.loss_chunk(lg[:n], c0, n, db.target_ids[c0:c0 + n], db.logp_behav[c0:c0 + n],
                        db.cu_seqlens, adv, inv, traj_sum, stats, dlogits=dl[:n], V=b.V)
    torch.cuda.synchronize()
    st = stats.cpu().numpy()
    # `stale` carries partial-rollout trajectories (C1 violations by design)
    assert vo.summary_dict()["valid"] == (0 if b.token_version is not None else 1)
    assert st[G.STAT_ROWS] == gold["T"]
    # loss within 1e-5 under the guarded criterion (Z17)
    err = abs(st[G.STAT_J] - gold["J"]) / max(abs(gold["J"]), 1e-2 * gold["S_abs"])
    assert err <= 1e-5, (st[G.STAT_J], gold["J"], err)
    assert abs(st[G.STAT_ABS] - gold["S_abs"]) <= 1e-5 * gold["S_abs"]
    assert abs(st[G.STAT_CLIPPED] - gold["n_clipped"]) <= gold["n_near_boundary"]
    assert abs(st[G.STAT_LOGP] - gold["sum_logp"]) <= 1e-6 * abs(gold["sum_logp"])
    ts = traj_sum.cpu().numpy()
    ref = np.array(gold["traj_sum"])
    L = np.diff(b.cu_seqlens)
    assert np.all(np.abs(ts - ref) <= 1e-5 * np.maximum(np.abs(ref), 1e-3 * L) + 1e-6)
