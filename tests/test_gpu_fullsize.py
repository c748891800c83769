"""-m gpu: parity at BASELINE.json's full sizes in the launch configuration bench.py
times (default plan, 131072-row resident chunk, V = 152064 / 262144), on sampled
rows the oracle computes one by one, plus properties that hold at any size."""
import numpy as np
import pytest
import torch

import oracle.oracle as O
import paper_2604_26256_b200 as G
import synth.gpu as SG
from synth.gen import bf16_bits_to_f32, make_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,R", [("prod", 131072), ("large", 32768), ("stale", 65536),
                                    ("dapo", 131072)])
def test_fullsize_chunk_sampled_rows(dev, name, R):
    b = make_batch(name, 0, period=R)
    V, ld = b.V, b.ld
    lg = torch.empty((R, ld), dtype=torch.int16, device=dev)
    dl = torch.empty_like(lg)
    SG.fill_logits(lg, b.logits, 0, R, V)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    vo = loss.validate(db)
    adv, inv = loss.advantage(db)
    T = b.T
    logp = torch.empty(T, device=dev)
    lse = torch.empty(T, device=dev)
    scale = torch.empty(T, device=dev)
    traj_sum = torch.zeros(b.N, dtype=torch.float64, device=dev)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    rng = np.random.default_rng(0)
    checks = []
    for c0 in range(0, T, R):
        n = min(R, T - c0)
        loss.loss_chunk(lg[:n], c0, n, db.target_ids[c0:c0 + n], db.logp_behav[c0:c0 + n],
                        db.cu_seqlens, adv, inv, traj_sum, stats, dlogits=dl[:n],
                        logp_out=logp[c0:c0 + n], lse_out=lse[c0:c0 + n],
                        scale_out=scale[c0:c0 + n], V=V)
        if c0 == 0 or c0 + R >= T:   # sample rows of the first and the last chunk
            ks = np.sort(rng.choice(n, size=12, replace=False))
            torch.cuda.synchronize()
            checks.append((c0, ks, dl[torch.from_numpy(ks).to(dev)].cpu().numpy().view(np.uint16)))
    torch.cuda.synchronize()
    summ = vo.summary_dict()
    assert summ["valid"] == (0 if b.token_version is not None else 1)
    adv_ref, inv_ref, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P, float(np.float32(1e-8)))
    assert np.array_equal(adv.cpu().numpy(), adv_ref.astype(np.float32))
    lp_h, lse_h, sc_h = logp.cpu().numpy(), lse.cpu().numpy(), scale.cpu().numpy()
    for c0, ks, dl_rows in checks:
        rows = c0 + ks
        bits = b.logits_bits(rows)           # logical row t reads physical row t % R
        rr = O.rows(rows, bits, V, b.target_ids[rows], b.logp_behav[rows], b.cu_seqlens, adv_ref,
                    inv_ref, 0.2, want_dlogits=True)
        assert np.max(np.abs(lp_h[rows] - rr.logp)) < 2e-3
        assert np.max(np.abs(lp_h[rows] - rr.logp)) < 1e-4      # fp32 is far inside the bound
        assert np.max(np.abs(lse_h[rows] - rr.lse)) < 1e-4
        got = bf16_bits_to_f32(dl_rows[:, :V]).astype(np.float64)
        den = np.linalg.norm(rr.dlogits)
        if den > 0:
            assert np.linalg.norm(got - rr.dlogits) / den < 1e-2
        for j in range(len(rows)):
            if rr.s[j] == 0.0 and abs(rr.r[j] - 1.2) > 1e-5 and abs(rr.r[j] - 0.8) > 1e-5:
                assert np.all(got[j] == 0.0)
            else:
                # properties at any size: the row sums to ~0 (bf16 rounding of the
                # non-target mass and of the target entry: <= 2 * 2^-9 * |s|) and the
                # target entry has sign -s
                assert abs(got[j].sum()) <= 2 * 2.0 ** -9 * abs(sc_h[rows[j]]) + 1e-30
                y = b.target_ids[rows[j]]
                assert np.sign(got[j, y]) == -np.sign(sc_h[rows[j]]) or got[j, y] == 0.0
    st = stats.cpu().numpy()
    assert st[G.STAT_ROWS] == T
    assert abs(st[G.STAT_J]) <= st[G.STAT_ABS]
    ts = traj_sum.cpu().numpy()
    assert abs(np.sum(inv_ref * ts) - st[G.STAT_J]) <= 1e-6 * st[G.STAT_ABS]


@pytest.mark.parametrize("world", [2, 4])
def test_vocab_parallel_fullsize_sampled_rows(dev, world):
    """NEXT(3) at the metric's size: a 65536-row chunk of `prod` (V = 152064) cut into `world`
    column shards, all ranks in one cooperative launch (the peer-memory protocol of the
    multi-GPU run), sampled rows against the oracle and the J invariants."""
    R = 65536
    b = make_batch("prod", 0, period=R)
    V, ld = b.V, b.ld
    lg = torch.empty((R, ld), dtype=torch.int16, device=dev)
    SG.fill_logits(lg, b.logits, 0, R, V)
    comm = G.VpGroup.local(world, V, R, dev)
    sc = comm.shard_cols
    shards = []
    for q in range(world):
        sh = torch.full((R, sc), 0x7FC1, dtype=torch.int16, device=dev)
        lo, hi = q * sc, min((q + 1) * sc, V)
        sh[:, :hi - lo] = lg[:, lo:hi]
        shards.append(sh)
    del lg
    dsh = [torch.empty_like(s) for s in shards]
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    logp = torch.empty(R, device=dev)
    scale = torch.empty(R, device=dev)
    ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
    st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    loss.loss_chunk_vp(comm, shards, 0, R, db.target_ids[:R], db.logp_behav[:R], db.cu_seqlens, adv,
                       inv, ts, st, dshards=dsh, logp_out=logp, scale_out=scale, V=V)
    torch.cuda.synchronize()
    adv_ref, inv_ref, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P, float(np.float32(1e-8)))
    rows = np.sort(np.random.default_rng(world).choice(R, size=12, replace=False))
    bits = b.logits_bits(rows)
    rr = O.rows(rows, bits, V, b.target_ids[rows], b.logp_behav[rows], b.cu_seqlens, adv_ref,
                inv_ref, 0.2, want_dlogits=True)
    r_idx = torch.from_numpy(rows).to(dev)
    assert np.max(np.abs(logp[r_idx].cpu().numpy() - rr.logp)) < 1e-4
    got = np.concatenate([bf16_bits_to_f32(d[r_idx].cpu().numpy().view(np.uint16)) for d in dsh],
                         axis=1)[:, :V].astype(np.float64)
    den = np.linalg.norm(rr.dlogits)
    assert np.linalg.norm(got - rr.dlogits) / den < 1e-2
    s = st.cpu().numpy()
    assert s[G.STAT_ROWS] == R and abs(s[G.STAT_J]) <= s[G.STAT_ABS]
