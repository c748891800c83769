"""-m gpu: advantages from sharded rewards (grpo_async_group_partials / _group_sq_partials /
_advantage_from_stats, the north_star "group reward statistics" all-reduce variant): R ranks
emulated in one process (each rank sees only its LPT share of the trajectories; the two
all-reduce rounds are a sum / max over the ranks' partials) against the fp64 oracle.
Synthetic rewards are 0/1, so every partial sum is exact and the result is bit-identical to
the single-rank oracle; continuous rewards agree to fp64 rounding."""
import numpy as np
import pytest
import torch

import oracle.oracle as O
import paper_2604_26256_b200 as G
from paper_2604_26256_b200 import _lib as L
from synth.gen import make_batch

pytestmark = pytest.mark.gpu


def _sharded(b, R, dev, rewards=None, norm=0, unbiased=False, mask=None, std_floor=1e-8):
    rew = np.asarray(b.rewards if rewards is None else rewards, np.float32)
    parts = G.lpt_partition(b.lengths, R)
    P = b.P
    local = []
    for ids in parts:
        L_loc = b.lengths[ids]
        cu = np.zeros(len(ids) + 1, np.int64)
        cu[1:] = np.cumsum(L_loc)
        t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to(dt).to(dev)
        local.append(dict(ids=ids, r=t(rew[ids], torch.float32), g=t(b.group_ids[ids], torch.int32),
                          cu=t(cu, torch.int64),
                          m=None if mask is None else t(mask[ids].astype(np.uint8), torch.uint8)))
    ps = []
    for d in local:
        part = torch.empty(4 * P + 1, dtype=torch.float64, device=dev)
        L.grpo_async_group_partials(d["r"], d["g"], d["cu"], len(d["ids"]), P, part, d["m"])
        ps.append(part)
    st = torch.stack(ps)
    glob = st.sum(0)
    p4 = st[:, :4 * P].view(R, P, 4)
    glob[:4 * P].view(P, 4)[:, 2:] = p4[:, :, 2:].max(0).values
    ss = torch.zeros(P, dtype=torch.float64, device=dev)
    for d in local:
        s = torch.empty(P, dtype=torch.float64, device=dev)
        L.grpo_async_group_sq_partials(d["r"], d["g"], len(d["ids"]), P, glob, s)
        ss += s
    adv = np.zeros(b.N, np.float32)
    inv = np.zeros(b.N, np.float32)
    for d in local:
        n = len(d["ids"])
        a = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        w = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        L.grpo_async_advantage_from_stats(d["r"], d["g"], d["cu"], n, P, std_floor, norm, d["m"],
                                          unbiased, glob, ss, a, w)
        adv[d["ids"]] = a.cpu().numpy()[:n]
        inv[d["ids"]] = w.cpu().numpy()[:n]
    torch.cuda.synchronize()
    return adv, inv


@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["tiny", "dapo", "prod"])
def test_sharded_advantages_bitexact(dev, name, R):
    b = make_batch(name, 0)
    adv, inv = _sharded(b, R, dev)
    ref_adv, ref_inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P,
                                      float(np.float32(1e-8)))
    assert np.array_equal(adv, ref_adv.astype(np.float32))
    assert np.array_equal(inv, ref_inv.astype(np.float32))


@pytest.mark.parametrize("R", [2, 4])
def test_sharded_advantages_options_and_continuous_rewards(dev, R):
    b = make_batch("dapo", 1)
    rng = np.random.default_rng(R)
    cont = rng.normal(size=b.N).astype(np.float32)
    mask = (rng.random(b.N) > 0.2)
    for norm, unb in ((0, False), (1, False), (0, True), (1, True)):
        adv, inv = _sharded(b, R, dev, rewards=cont, norm=norm, unbiased=unb, mask=mask)
        ref_adv, _, gc = O.advantage(cont, b.group_ids, b.cu_seqlens, b.P, float(np.float32(1e-8)),
                                     unbiased=unb)
        ref_inv = O.weights(b.group_ids, b.cu_seqlens, gc, b.P, norm, mask.astype(np.uint8))
        np.testing.assert_allclose(adv, ref_adv, rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(inv, ref_inv, rtol=1e-6, atol=0)
    # a bitwise-equal group keeps A = 0 exactly across ranks
    eq = cont.copy()
    eq[b.group_ids == 0] = np.float32(0.3)
    adv, _ = _sharded(b, R, dev, rewards=eq)
    assert np.all(adv[b.group_ids == 0] == 0.0)
