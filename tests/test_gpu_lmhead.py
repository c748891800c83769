"""-m gpu: NEXT(2) -- the LM-head-fused loss (tcgen05 GEMM X W^T with the loss in its
epilogue; backward: recomputed logits -> dz in the epilogue, then dX = dz W and
dW += dz^T X) against the fp64 oracle (oracle.run_batch_lmhead).

Tolerances: BASELINE north_star -- logp 2e-3 absolute, J 1e-5 relative (guarded at
1e-2 * S_abs, Z17), dz / dX / dW 1e-2 relative L2.  The logits are fp32 tensor-core
sums of d bf16 products rather than exact bf16 inputs, so J may also move by the propagated
a-priori bound of that accumulation (Z25, tests/gpu_util.lmhead_accum_J_bound,
computed from X and W alone); measured logp errors are 3-6e-6."""
import numpy as np
import pytest
import torch

import oracle.oracle as O
import paper_2604_26256_b200 as G
from synth.gen import make_batch
from paper_2604_26256_b200 import _lib as L
from tests.gpu_util import compare, lmhead_accum_J_bound, lmhead_batch, run_gpu_lmhead, to_dev_bits

pytestmark = pytest.mark.gpu


def _rel_l2(a, b):
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a))


def _check(gpu, ref, b, X, W, eps_hi=None):
    errs = compare(gpu, ref, b, loss_rtol=1e-5, eps_hi=eps_hi,
                   extra_J_tol=lmhead_accum_J_bound(b, X, W, ref))
    assert gpu["dz_pad_untouched"]
    errs["dhidden_rel_l2"] = _rel_l2(gpu["dhidden"], ref["dhidden"])
    errs["dW_rel_l2"] = _rel_l2(gpu["dW"], ref["dW"])
    assert errs["dhidden_rel_l2"] <= 1e-2, errs
    assert errs["dW_rel_l2"] <= 1e-2, errs
    return errs


@pytest.mark.parametrize("d", [64, 256])
@pytest.mark.parametrize("name", ["tiny", "ragged", "mid32k"])
def test_lmhead_parity(dev, name, d, cta_group):
    b, X, W = lmhead_batch(name, 3, d)
    ref = O.run_batch_lmhead(b, X, W, std_floor=float(np.float32(1e-8)))
    gpu = run_gpu_lmhead(b, X, W, dev)
    errs = _check(gpu, ref, b, X, W)
    print(name, d, errs)


def test_lmhead_parity_152k_chunked(dev, cta_group):
    """The metric's vocabulary (V = 152064, 594 tiles of 256) with row chunks that are not
    multiples of the 128-row tile."""
    b, X, W = lmhead_batch("mid152k", 4, 128)
    ref = O.run_batch_lmhead(b, X, W, std_floor=float(np.float32(1e-8)))
    gpu = run_gpu_lmhead(b, X, W, dev, chunks=3)
    print(_check(gpu, ref, b, X, W))


def test_lmhead_dapo_options(dev):
    b, X, W = lmhead_batch("ragged", 5, 128)
    mask = (b.lengths < np.percentile(b.lengths, 80)).astype(np.uint8)
    ref = O.run_batch_lmhead(b, X, W, std_floor=float(np.float32(1e-8)), eps_hi=0.28, norm=1,
                             traj_mask=mask)
    gpu = run_gpu_lmhead(b, X, W, dev, eps_hi=0.28, norm="token", traj_mask=mask)
    _check(gpu, ref, b, X, W, eps_hi=0.28)


@pytest.fixture(params=[1, 2], ids=["cg1", "cg2"])
def cta_group(request):
    L.grpo_async_lmhead_set_cta_group(request.param)
    yield request.param
    L.grpo_async_lmhead_set_cta_group(2)


@pytest.mark.parametrize("shape", [(1, 64, 1), (127, 64, 255), (129, 128, 257), (300, 192, 1000),
                                   (513, 256, 4099)])
def test_lmhead_logits_gemm(dev, shape, cta_group):
    """The tcgen05 GEMM alone (ragged n, V; minimum d) against the fp64 product: every
    logit within half a bf16 ulp plus the fp32 accumulation bound d * 2^-23 * sum|x w|."""
    n, d, V = shape
    rng = np.random.default_rng(n + d + V)
    from synth.gen import f32_to_bf16_bits
    X = f32_to_bf16_bits(rng.standard_normal((n, d), dtype=np.float32))
    W = f32_to_bf16_bits(rng.standard_normal((V, d), dtype=np.float32) * np.float32(0.2))
    ld = (V + 7) // 8 * 8 + 8
    out = torch.full((n, ld), 0x7FC3, dtype=torch.int16, device=dev)
    L.grpo_async_lmhead_logits(to_dev_bits(X, dev).view(torch.bfloat16),
                               to_dev_bits(W, dev).view(torch.bfloat16), n, d, V,
                               out.view(torch.bfloat16), ld)
    torch.cuda.synchronize()
    raw = out.cpu().numpy().view(np.uint16)
    got = O._bf16_to_f64(raw[:, :V])
    z = O.lmhead_logits(X, W)
    bound = np.abs(O._bf16_to_f64(X)) @ np.abs(O._bf16_to_f64(W)).T * d * 2.0 ** -23
    assert np.all(np.abs(got - z) <= np.abs(z) * 2.0 ** -8 + bound)
    assert np.all(raw[:, V:] == 0x7FC3)


def test_lmhead_fused_matches_unfused(dev):
    """lmhead_fwd (logits never stored) against lmhead_logits -> loss_chunk on the stored
    bf16 logits: same per-row logp within the bf16 rounding of the stored logits."""
    b, X, W = lmhead_batch("mid32k", 6, 128)
    gpu = run_gpu_lmhead(b, X, W, dev, want_grads=False)
    Xd = to_dev_bits(X, dev).view(torch.bfloat16)
    Wd = to_dev_bits(W, dev).view(torch.bfloat16)
    ld = b.ld
    lg = torch.zeros((b.T, ld), dtype=torch.bfloat16, device=dev)
    L.grpo_async_lmhead_logits(Xd, Wd, b.T, X.shape[1], b.V, lg, ld)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    logp = torch.empty(b.T, device=dev)
    ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
    st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    loss.loss_chunk(lg, 0, b.T, db.target_ids, db.logp_behav, db.cu_seqlens, adv, inv, ts, st,
                    logp_out=logp, V=b.V)
    torch.cuda.synchronize()
    assert np.max(np.abs(logp.cpu().numpy() - gpu["logp"])) < 0.05


def test_lmhead_bad_args(dev):
    W = torch.zeros((10, 96), dtype=torch.bfloat16, device=dev)
    X = torch.zeros((4, 96), dtype=torch.bfloat16, device=dev)
    out = torch.zeros((4, 16), dtype=torch.bfloat16, device=dev)
    with pytest.raises(L.GrpoError) as e:
        L.grpo_async_lmhead_logits(X, W, 4, 96, 10, out, 16)  # d % 64 != 0
    assert e.value.status == L.GRPO_ERR_INVALID_ARG


def _run_tp(b, X, W, dev, R, chunks=1):
    """Tensor-parallel LM head with R vocabulary shards emulated in one process: all-gather =
    stacking the shards' row partials, all-reduce = summing their dhidden partials."""
    T, V = b.T, b.V
    d = X.shape[1]
    Vs = -(-V // R)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    loss.validate(db)
    adv, inv = loss.advantage(db)
    Xd = to_dev_bits(X, dev).view(torch.bfloat16)
    Wd = to_dev_bits(W, dev).view(torch.bfloat16)
    shards = [(q * Vs, Wd[q * Vs:min((q + 1) * Vs, V)].contiguous()) for q in range(R)]
    logp = torch.full((T,), float("nan"), device=dev)
    lse = torch.full((T,), float("nan"), device=dev)
    scale = torch.full((T,), float("nan"), device=dev)
    traj_sum = torch.zeros(b.N, dtype=torch.float64, device=dev)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    dX = torch.zeros((T, d), dtype=torch.float32, device=dev)
    dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
    dz_full = np.zeros((T, V), np.float64)
    bounds = np.linspace(0, T, chunks + 1).astype(np.int64)
    for c in range(chunks):
        r0, r1 = int(bounds[c]), int(bounds[c + 1])
        n = r1 - r0
        parts = []
        for off, Wq in shards:
            ws = torch.empty(L.grpo_async_lmhead_workspace_size(n, Wq.shape[0], 1), dtype=torch.uint8,
                             device=dev)
            part = torch.empty((max(n, 1), 4), dtype=torch.float32, device=dev)
            L.grpo_async_lmhead_tp_partials(Xd[r0:r1], Wq, n, d, Wq.shape[0], off,
                                            db.target_ids[r0:r1], part, ws)
            parts.append(part)
        loss.lmhead_tp_fwd(Xd[r0:r1], shards[0][1], 0, V, r0, n, db.target_ids[r0:r1],
                           db.logp_behav[r0:r1], db.cu_seqlens, adv, inv, traj_sum, stats,
                           allgather=lambda t, parts=parts: torch.stack(parts),
                           logp_out=logp[r0:r1], lse_out=lse[r0:r1], scale_out=scale[r0:r1])
        for off, Wq in shards:
            Vq = Wq.shape[0]
            ld = (Vq + 7) // 8 * 8
            dz = torch.zeros((n, ld), dtype=torch.bfloat16, device=dev)
            dpart = torch.empty((n, d), dtype=torch.float32, device=dev)
            loss.lmhead_tp_bwd(Xd[r0:r1], Wq, off, n, db.target_ids[r0:r1], lse[r0:r1],
                               scale[r0:r1], dz, dhidden_partial=dpart, dW_shard=dW[off:off + Vq])
            dX[r0:r1] += dpart
            dz_full[r0:r1, off:off + Vq] = dz[:, :Vq].float().cpu().numpy()
    torch.cuda.synchronize()
    return dict(logp=logp.cpu().numpy().astype(np.float64), lse=lse.cpu().numpy().astype(np.float64),
                scale=scale.cpu().numpy().astype(np.float64), stats=stats.cpu().numpy(),
                traj_sum=traj_sum.cpu().numpy(), dz=dz_full, dX=dX.cpu().numpy().astype(np.float64),
                dW=dW.cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("R", [1, 2, 3, 4])
@pytest.mark.parametrize("name,d", [("ragged", 128), ("mid32k", 64)])
def test_lmhead_tensor_parallel(dev, name, d, R, cta_group):
    """NEXT(2) x NEXT(3): W split by vocabulary rows over R ranks (uneven last shard), per-row
    partials combined in rank order, dhidden partials summed -- against the oracle on the
    whole W (same tolerances as the single-GPU LM head)."""
    b, X, W = lmhead_batch(name, 7, d)
    ref = O.run_batch_lmhead(b, X, W, std_floor=float(np.float32(1e-8)))
    g = _run_tp(b, X, W, dev, R, chunks=2)
    rr = ref["rows"]
    assert np.max(np.abs(g["logp"] - rr.logp)) <= 2e-3
    S_abs = float(np.sum(ref["inv_norm"][np.repeat(np.arange(b.N), b.lengths)] * np.abs(rr.term)))
    J = g["stats"][G.STAT_J]
    # DESIGN.md Z17 guard plus the tensor cores' accumulation bound (Z25)
    assert abs(J - ref["J"]) <= 1e-5 * max(abs(ref["J"]), 1e-2 * S_abs) + lmhead_accum_J_bound(b, X, W, ref)
    for k, rk in (("dz", rr.dlogits), ("dX", ref["dhidden"]), ("dW", ref["dW"])):
        assert _rel_l2(g[k], rk) <= 1e-2, k


@pytest.mark.parametrize("cg", [2])
def test_lmhead_fullsize_sampled_rows(dev, cg):
    """The LM-head bench workload at full size (8190 rows of `prod`, d = 5120, V = 152064) in
    the launch configuration scripts/bench_lmhead.py times, checked on 12 sampled rows that
    the oracle computes one by one: logp, lse, token scale, the dz row and the dX row."""
    import dataclasses

    from synth.gen import lmhead_inputs
    L.grpo_async_lmhead_set_cta_group(cg)
    b0 = make_batch("prod", 0)
    n = int(b0.cu_seqlens[int(np.searchsorted(b0.cu_seqlens, 8192, side="right") - 1)])
    d, V = 5120, b0.V
    X, W = lmhead_inputs(n, V, d, 11)
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(n, 12, replace=False))
    z = O.lmhead_logits_rows(X[rows], W)
    m = z.max(1, keepdims=True)
    lse_rows = (m + np.log(np.exp(z - m).sum(1, keepdims=True)))[:, 0]
    tgt = b0.target_ids[:n]
    logp_rows = z[np.arange(len(rows)), tgt[rows]] - lse_rows
    # test-side inputs: behaviour log-probs of the sampled rows near the oracle's own logp
    lw = np.array(b0.logp_behav[:n], np.float32)
    lw[rows] = (logp_rows - rng.normal(size=len(rows)) * 0.05).astype(np.float32)
    full_lw = np.array(b0.logp_behav, np.float32)
    full_lw[:n] = lw
    b = dataclasses.replace(b0, logp_behav=full_lw)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    Xd = to_dev_bits(X, dev).view(torch.bfloat16)
    Wd = to_dev_bits(W, dev).view(torch.bfloat16)
    logp = torch.empty(n, device=dev)
    lse = torch.empty(n, device=dev)
    scale = torch.empty(n, device=dev)
    ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
    st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    loss.lmhead_fwd(Xd, Wd, 0, n, db.target_ids[:n], db.logp_behav[:n], db.cu_seqlens, adv, inv, ts,
                    st, logp_out=logp, lse_out=lse, scale_out=scale)
    dz = torch.empty((n, V), dtype=torch.bfloat16, device=dev)
    dX = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
    loss.lmhead_bwd(Xd, Wd, n, db.target_ids[:n], lse, scale, dz, dhidden=dX)
    torch.cuda.synchronize()
    ref_adv, ref_inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P, float(np.float32(1e-8)))
    rr = O.rows_f64(rows, z, tgt[rows], lw[rows], b.cu_seqlens, ref_adv, ref_inv, 0.2)  # row-local
    r_idx = torch.from_numpy(rows).to(dev)
    g_logp = logp[r_idx].cpu().numpy()
    assert np.max(np.abs(g_logp - rr.logp)) <= 2e-3
    assert np.max(np.abs(lse[r_idx].cpu().numpy() - rr.lse)) <= 2e-3
    assert np.allclose(scale[r_idx].cpu().numpy(), rr.s, rtol=1e-3, atol=1e-12)
    g_dz = dz[r_idx].float().cpu().numpy().astype(np.float64)
    assert _rel_l2(g_dz, rr.dlogits) <= 1e-2
    ref_dX = O.matmul_rows_W(rr.dlogits, W)
    assert _rel_l2(dX[r_idx].float().cpu().numpy().astype(np.float64), ref_dX) <= 1e-2
    L.grpo_async_lmhead_set_cta_group(2)


@pytest.mark.parametrize("R", [1, 2, 3, 4])
@pytest.mark.parametrize("name,d", [("ragged", 128), ("mid32k", 256)])
def test_lmhead_tp_dx_gemm_reduce_scatter(dev, name, d, R):
    """grpo_async_lmhead_tp_dx: dz_q W_q on the tensor cores (B read MN-major from the
    row-major W shard) with the f32 tiles stored straight into the owner rank's slot; then
    the owner's rank-order sum.  R ranks emulated on one GPU (the slot buffers are local).
    Against the oracle's dhidden and against the plain dX GEMM's partials summed."""
    b, X, W = lmhead_batch(name, 9, d)
    ref = O.run_batch_lmhead(b, X, W, std_floor=float(np.float32(1e-8)))
    T, V = b.T, b.V
    Vs = -(-V // R)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    Xd = to_dev_bits(X, dev).view(torch.bfloat16)
    Wd = to_dev_bits(W, dev).view(torch.bfloat16)
    lse = torch.empty(T, device=dev)
    scale = torch.empty(T, device=dev)
    ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
    st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    loss.lmhead_fwd(Xd, Wd, 0, T, db.target_ids, db.logp_behav, db.cu_seqlens, adv, inv, ts, st,
                    lse_out=lse, scale_out=scale)
    rpr = -(-T // R)
    # two halves per slot buffer; call e writes half e % 2 (epoch double buffering)
    bufs = [torch.full((2, R, rpr, d), float("nan"), device=dev) for _ in range(R)]
    gemm_sum = torch.zeros((T, d), device=dev)
    dzs = []
    for q in range(R):
        off = q * Vs
        Wq = Wd[off:min(off + Vs, V)].contiguous()
        Vq = Wq.shape[0]
        ld = (Vq + 7) // 8 * 8
        dz = torch.zeros((T, ld), dtype=torch.bfloat16, device=dev)
        part = torch.empty((T, d), device=dev)
        loss.lmhead_tp_bwd(Xd, Wq, off, T, db.target_ids, lse, scale, dz, dhidden_partial=part)
        gemm_sum += part
        dzs.append((dz, ld, Wq, Vq))
    for epoch in (1, 0):
        for q, (dz, ld, Wq, Vq) in enumerate(dzs):
            L.grpo_async_lmhead_tp_dx(dz, ld, Wq, T, d, Vq, R, q, bufs, epoch)
        if epoch == 1:  # the other half is untouched
            torch.cuda.synchronize()
            assert all(torch.isnan(b_[0]).all().item() for b_ in bufs)
        outs = []
        for q in range(R):
            rows = max(0, min(rpr, T - q * rpr))
            o = torch.empty((max(rows, 1), d), device=dev)
            L.grpo_async_lmhead_tp_dx_reduce(bufs[q], R, T, d, q, o, epoch)
            outs.append(o[:rows])
        torch.cuda.synchronize()
        dX = torch.cat(outs).cpu().numpy().astype(np.float64)
        assert dX.shape == (T, d) and np.isfinite(dX).all()
        assert _rel_l2(dX, ref["dhidden"]) <= 1e-2
        # two f32 GEMMs (the plain dX GEMM per shard, summed; the fused one) in different orders
        assert _rel_l2(dX, gemm_sum.cpu().numpy().astype(np.float64)) <= 1e-3


@pytest.mark.parametrize("seed", range(6))
def test_lmhead_random_shapes(dev, seed, cta_group):
    """Fuzz: random row count (ragged 128/256-row tiles), d (multiples of 64), V (ragged 256
    tiles) and chunking for the fused forward + backward against the oracle."""
    import dataclasses

    from synth.gen import lmhead_inputs
    rng = np.random.default_rng(900 + seed)
    d = 64 * int(rng.integers(1, 7))
    V = int(rng.integers(3, 5000))
    base = make_batch("ragged", seed)
    b = dataclasses.replace(base, V=V, ld=(V + 7) // 8 * 8,
                            target_ids=(base.target_ids % V).astype(np.int64))
    X, W = lmhead_inputs(b.T, V, d, seed)
    z = O.lmhead_logits(X, W)
    m = z.max(1, keepdims=True)
    lse = (m + np.log(np.exp(z - m).sum(1, keepdims=True)))[:, 0]
    lw = (z[np.arange(b.T), b.target_ids] - lse - rng.normal(size=b.T) * 0.05).astype(np.float32)
    b = dataclasses.replace(b, logp_behav=lw)
    ref = O.run_batch_lmhead(b, X, W, std_floor=float(np.float32(1e-8)))
    gpu = run_gpu_lmhead(b, X, W, dev, chunks=int(rng.integers(1, 4)))
    _check(gpu, ref, b, X, W)


def test_lmhead_dynamic_units_concurrent_streams(dev):
    """The dynamic unit counters (csrc/sched.cuh): 96 LM-head GEMM launches -- logits (forward
    kernel) and dW (gemm_kernel) -- spread over four streams at once, more launches than the
    64 counter slots, each result bit-identical to the same launch run alone.  A counter
    shared by two running launches or not zeroed would drop or repeat units."""
    n, d, V = 700, 128, 3001
    rng = np.random.default_rng(7)
    from synth.gen import f32_to_bf16_bits
    X = to_dev_bits(f32_to_bf16_bits(rng.standard_normal((n, d), dtype=np.float32)), dev).view(torch.bfloat16)
    W = to_dev_bits(f32_to_bf16_bits(rng.standard_normal((V, d), dtype=np.float32) * np.float32(0.2)),
                    dev).view(torch.bfloat16)
    ld = (V + 7) // 8 * 8
    ref = torch.empty((n, ld), dtype=torch.bfloat16, device=dev)
    L.grpo_async_lmhead_logits(X, W, n, d, V, ref, ld)
    dW_ref = torch.zeros((V, d), dtype=torch.float32, device=dev)
    L.grpo_async_lmhead_dw(X, n, d, V, ref, ld, dW_ref)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(device=dev) for _ in range(4)]
    outs = [torch.empty((n, ld), dtype=torch.bfloat16, device=dev) for _ in range(48)]
    dws = [torch.zeros((V, d), dtype=torch.float32, device=dev) for _ in range(48)]
    for k in range(48):
        s = streams[k % 4]
        L.grpo_async_lmhead_logits(X, W, n, d, V, outs[k], ld, stream=s)
        L.grpo_async_lmhead_dw(X, n, d, V, ref, ld, dws[k], stream=s)
    torch.cuda.synchronize()
    for k in range(48):
        assert torch.equal(outs[k][:, :V], ref[:, :V]), k
        assert torch.equal(dws[k], dW_ref), k
