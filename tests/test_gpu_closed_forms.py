"""-m gpu: the closed forms HW4 and HW5 (pinned on the oracle at small size in
tests/test_oracle_pins.py) at BASELINE.json's full sizes through the launch configuration
bench.py times -- the whole `prod` batch (1,008,179 rows, V = 152064, 131072-row chunks, the
auto plan K3c stream_kernel<512,1,2048,1>) and `large` (2.17M rows, V = 262144, rows split
over two-SM clusters).  Every logits row is uniform (all zeros), so log pi_theta(y_t) =
-ln V exactly for any target and the objective has a closed form:

  HW4  constant ratio r = exp(-ln V - logp_w) > 1 + eps on every token (eq:grpo_async P:9-26,
       clip P:151): positive-advantage tokens clip, the others do not, and
       J = (1/P) sum_p S_p+ (1 + eps - r) / G_p,   S_p+ = sum of the group's positive A_i
       (eq:group_advantage P:153-156);
  HW5  on-policy, logp_w = logp_theta: r = 1 and J = 0, advantages being zero-mean per group.

The dlogits of a uniform row are s_t (1/V - [v = y_t]): checked on sampled rows of every
chunk, with the clipped rows exactly zero."""
import math

import numpy as np
import pytest
import torch

import oracle.oracle as O
import paper_2604_26256_b200 as G
from synth.gen import bf16_bits_to_f32, make_batch

pytestmark = pytest.mark.gpu
EPS = float(np.float32(0.2))


def _run_uniform(dev, b, lw, R):
    """bench.py's step on all-zero logits with behaviour log-probs lw: stats and sampled
    rows (index, token scale, dlogits row) of every chunk."""
    import dataclasses
    b = dataclasses.replace(b, logp_behav=lw)
    lg = torch.zeros((R, b.ld), dtype=torch.int16, device=dev)
    dl = torch.empty_like(lg)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    vo = loss.validate(db)
    adv, inv = loss.advantage(db)
    scale = torch.empty(b.T, device=dev)
    logp = torch.empty(b.T, device=dev)
    traj_sum = torch.zeros(b.N, dtype=torch.float64, device=dev)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    rng = np.random.default_rng(1)
    samples = []
    for c0 in range(0, b.T, R):
        n = min(R, b.T - c0)
        loss.loss_chunk(lg[:n], c0, n, db.target_ids[c0:c0 + n], db.logp_behav[c0:c0 + n],
                        db.cu_seqlens, adv, inv, traj_sum, stats, dlogits=dl[:n],
                        scale_out=scale[c0:c0 + n], logp_out=logp[c0:c0 + n], V=b.V)
        ks = np.sort(rng.choice(n, size=4, replace=False))
        rows_dl = dl[torch.from_numpy(ks).to(dev)].cpu().numpy().view(np.uint16)[:, :b.V]
        samples.append((c0 + ks, rows_dl))
    plan = G.grpo_async_last_plan()
    torch.cuda.synchronize()
    return dict(stats=stats.cpu().numpy(), scale=scale.cpu().numpy(), logp=logp.cpu().numpy(),
                summary=vo.summary_dict(), samples=samples, plan=plan, b=b)


def _check_uniform_rows(out, V):
    b = out["b"]
    for rows, dl_bits in out["samples"]:
        got = bf16_bits_to_f32(dl_bits).astype(np.float64)
        for j, t in enumerate(rows):
            s = float(out["scale"][t])
            y = int(b.target_ids[t])
            if s == 0.0:
                assert np.all(got[j] == 0.0)
                continue
            other = np.delete(got[j], y)
            assert np.all(other == other[0])                  # one value off the target
            assert abs(other[0] - s / V) <= 2.0 ** -8 * abs(s / V)
            assert abs(got[j, y] - s * (1.0 / V - 1.0)) <= 2.0 ** -8 * abs(s)


@pytest.mark.parametrize("name,R,kernel", [("prod", 131072, 3), ("large", 65536, 3)])
def test_hw4_constant_ratio_fullsize(dev, name, R, kernel):
    b = make_batch(name, 0, period=R)
    V = b.V
    lw = np.full(b.T, -math.log(V) - math.log(1.5), np.float32)
    out = _run_uniform(dev, b, lw, R)
    assert out["plan"]["kernel"] == kernel
    if V >= 200000:
        assert out["plan"]["cluster_size"] == 2      # the split-row plan of `large`
    # log pi_theta = -ln V on every row (fp32 output of the fp64 value)
    assert np.all(out["logp"] == np.float32(-math.log(V)))
    r = math.exp(-math.log(V) - float(np.float32(lw[0])))
    assert r > 1.0 + EPS
    adv, inv, gc = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P, float(np.float32(1e-8)))
    S_plus = np.zeros(b.P)
    np.add.at(S_plus, b.group_ids, np.where(adv > 0, adv, 0.0))
    J_closed = float(np.sum(S_plus * (1.0 + EPS - r) / gc) / b.P)
    st = out["stats"]
    S_abs = st[G.STAT_ABS]
    assert abs(st[G.STAT_J] - J_closed) <= 1e-5 * max(abs(J_closed), 1e-2 * S_abs), (st[G.STAT_J], J_closed)
    assert st[G.STAT_ROWS] == b.T
    # every token of a positive-advantage trajectory clips, and only those
    n_pos = int(np.sum(np.repeat(adv > 0, b.lengths)))
    assert st[G.STAT_CLIPPED] == n_pos
    _check_uniform_rows(out, V)


@pytest.mark.parametrize("name,R", [("prod", 131072), ("large", 65536)])
def test_hw5_on_policy_fullsize(dev, name, R):
    b = make_batch(name, 0, period=R)
    V = b.V
    lw = np.full(b.T, -math.log(V), np.float32)
    out = _run_uniform(dev, b, lw, R)
    st = out["stats"]
    assert st[G.STAT_CLIPPED] == 0
    # J = 0 exactly in exact arithmetic; the f32 advantages' rounding leaves ~1e-8 of S_abs
    assert abs(st[G.STAT_J]) <= 1e-5 * 1e-2 * st[G.STAT_ABS], (st[G.STAT_J], st[G.STAT_ABS])
    _check_uniform_rows(out, V)
