"""Helpers shared by the -m gpu parity tests: run the CUDA path through the C ABI
and the fp64 oracle on the same seeded inputs, and compare them under the
tolerances of BASELINE.json north_star / DESIGN.md "Parity"."""
from __future__ import annotations

import numpy as np
import torch

import oracle.oracle as O
import paper_2604_26256_b200 as G
from synth.gen import bf16_bits_to_f32

EPS32 = float(np.float32(0.2))
# DESIGN.md Z17: the relative loss criterion is taken against
# max(|J|, Z17_GUARD * S_abs), S_abs = sum_t inv_norm_i |term_t| the L1 mass of J's summands
Z17_GUARD = 1e-2


def to_dev_bits(bits: np.ndarray, device) -> torch.Tensor:
    """uint16 numpy bf16 bit patterns -> int16 CUDA tensor (same bits)."""
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(device)


def dev_bits_to_f64(t: torch.Tensor, V: int) -> np.ndarray:
    b = t.cpu().numpy().view(np.uint16)[:, :V]
    return bf16_bits_to_f32(b).astype(np.float64)


def run_gpu(batch, logits_bits, device, tune=None, chunks=1, inplace=False, want_dlogits=True,
            grad_scale=1.0, eps=0.2, eps_hi=None, norm="seq", traj_mask=None, std_unbiased=False):
    """Whole path on the GPU: validate, advantage, fused loss over `chunks` row chunks."""
    db = G.DeviceBatch.from_host(batch, device)
    mask_d = None if traj_mask is None else torch.from_numpy(
        np.ascontiguousarray(traj_mask, np.uint8)).to(device)
    loss = G.GrpoAsyncLoss(eps=eps, grad_scale=grad_scale, tune=tune, eps_hi=eps_hi, norm=norm,
                           traj_mask=mask_d, std_unbiased=std_unbiased)
    vo = loss.validate(db)
    adv, inv = loss.advantage(db)
    T, ld, V = batch.T, batch.ld, batch.V
    lg = to_dev_bits(logits_bits, device)
    assert lg.shape == (T, ld)
    dl = None
    if want_dlogits:
        dl = lg if inplace else torch.full((T, ld), 0x7FC3, dtype=torch.int16, device=device)
    logp = torch.full((T,), float("nan"), device=device)
    lse = torch.full((T,), float("nan"), device=device)
    scale = torch.full((T,), float("nan"), device=device)
    traj_sum = torch.zeros(batch.N, dtype=torch.float64, device=device)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=device)
    bounds = np.linspace(0, T, chunks + 1).astype(np.int64)
    for c in range(chunks):
        b, e = int(bounds[c]), int(bounds[c + 1])
        loss.loss_chunk(lg[b:e] if e > b else lg[:0], b, e - b, db.target_ids[b:e],
                        db.logp_behav[b:e], db.cu_seqlens, adv, inv, traj_sum, stats,
                        dlogits=(dl[b:e] if dl is not None else None), logp_out=logp[b:e],
                        lse_out=lse[b:e], scale_out=scale[b:e], V=V)
    torch.cuda.synchronize()
    out = dict(
        traj_flags=vo.traj_flags.cpu().numpy().view(np.uint32)[:batch.N],
        group_count=vo.group_count.cpu().numpy(),
        stale_hist=vo.stale_hist.cpu().numpy().reshape(batch.P, batch.K + 1),
        summary=vo.summary_dict(),
        adv=adv.cpu().numpy(), inv_norm=inv.cpu().numpy(),
        logp=logp.cpu().numpy().astype(np.float64), lse=lse.cpu().numpy().astype(np.float64),
        scale=scale.cpu().numpy().astype(np.float64),
        traj_sum=traj_sum.cpu().numpy(), stats=stats.cpu().numpy(),
        launches=loss.launches, inplace=inplace)
    if want_dlogits:
        out["dlogits_raw"] = dl.cpu().numpy().view(np.uint16)
        out["dlogits"] = bf16_bits_to_f32(out["dlogits_raw"][:, :V]).astype(np.float64)
    return out


def run_oracle(batch, logits_bits, want_dlogits=True, eps=0.2, grad_scale=1.0, eps_hi=None,
               norm="seq", traj_mask=None, std_unbiased=False):
    return O.run_batch(batch, logits_bits, eps=eps, grad_scale=grad_scale,
                       std_floor=float(np.float32(1e-8)), want_dlogits=want_dlogits,
                       eps_hi=eps_hi, norm={"seq": 0, "token": 1}[norm], traj_mask=traj_mask,
                       std_unbiased=std_unbiased)


def near_boundary(r, eps=EPS32, tol=1e-5, eps_hi=None):
    hi = eps if eps_hi is None else float(np.float32(eps_hi))
    return (np.abs(r - (1 + hi)) <= tol) | (np.abs(r - (1 - eps)) <= tol)


def compare(gpu, ref, batch, check_dlogits=True, logp_atol=2e-3, loss_rtol=1e-5, dl_rel=1e-2,
            logits_pad=None, eps_hi=None, extra_J_tol=0.0):
    """Assert the north_star criteria; returns a dict of measured errors."""
    rr = ref["rows"]
    errs = {}
    # bit-exact integer outputs
    assert np.array_equal(gpu["traj_flags"], ref["validate"]["traj_flags"]), "traj_flags"
    assert np.array_equal(gpu["group_count"], ref["validate"]["group_count"]), "group_count"
    assert np.array_equal(gpu["stale_hist"], ref["validate"]["stale_hist"]), "stale_hist"
    assert gpu["summary"] == ref["validate"]["summary"], (gpu["summary"], ref["validate"]["summary"])
    # advantages: same fp64 order -> identical after rounding to f32
    assert np.array_equal(gpu["adv"], ref["adv"].astype(np.float32)), "adv"
    assert np.array_equal(gpu["inv_norm"], ref["inv_norm"].astype(np.float32)), "inv_norm"
    # per-token log-probs
    errs["logp_max_abs"] = float(np.max(np.abs(gpu["logp"] - rr.logp))) if batch.T else 0.0
    assert errs["logp_max_abs"] <= logp_atol, errs
    errs["lse_max_abs"] = float(np.max(np.abs(gpu["lse"] - rr.lse))) if batch.T else 0.0
    assert errs["lse_max_abs"] <= logp_atol
    # loss (guarded relative criterion, Z17)
    J_ref = ref["J"]
    S_abs = float(np.sum(ref["inv_norm"][np.repeat(np.arange(batch.N), batch.lengths)] *
                         np.abs(rr.term)))
    J_gpu = gpu["stats"][G.STAT_J]
    errs["J_ref"], errs["J_gpu"] = J_ref, J_gpu
    errs["J_rel_guarded"] = abs(J_gpu - J_ref) / max(abs(J_ref), Z17_GUARD * S_abs, 1e-300)
    errs["J_rel_raw"] = abs(J_gpu - J_ref) / max(abs(J_ref), 1e-300)
    if extra_J_tol:  # the LM head's logits error (Z25), propagated into J
        errs["J_extra_tol"] = extra_J_tol
        assert abs(J_gpu - J_ref) <= loss_rtol * max(abs(J_ref), Z17_GUARD * S_abs) + extra_J_tol, errs
    else:
        assert errs["J_rel_guarded"] <= loss_rtol, errs
    assert abs(gpu["stats"][G.STAT_ABS] - S_abs) <= 1e-5 * S_abs + 1e-300
    # per-trajectory sums of terms (fp64 reductions of fp32 terms)
    ts_scale = np.maximum(np.abs(ref["traj_sum"]), 1e-3 * batch.lengths)
    assert np.all(np.abs(gpu["traj_sum"] - ref["traj_sum"]) <= 1e-5 * ts_scale + 1e-6), "traj_sum"
    # clip decisions: fp32 vs fp64 may differ only within 1e-5 of a clip boundary
    nb = near_boundary(rr.r, eps_hi=eps_hi)
    clipped_gpu_s = gpu["scale"] == 0.0
    oracle_zero_s = rr.s == 0.0
    mism = (clipped_gpu_s != oracle_zero_s) & ~nb
    assert not mism.any(), f"{mism.sum()} clip decisions differ away from a boundary"
    errs["boundary_flips"] = int(((clipped_gpu_s != oracle_zero_s) & nb).sum())
    assert abs(gpu["stats"][G.STAT_CLIPPED] - ref["n_clipped"]) <= errs["boundary_flips"]
    assert gpu["stats"][G.STAT_ROWS] == batch.T
    # token scale s_t (fp32) vs oracle
    ok_s = ~nb
    if ok_s.any():
        ds = np.abs(gpu["scale"][ok_s] - rr.s[ok_s])
        errs["scale_max_rel"] = float(np.max(ds / np.maximum(np.abs(rr.s[ok_s]), 1e-30)))
        assert np.all(ds <= 1e-4 * np.abs(rr.s[ok_s]) + 1e-12)
    if check_dlogits and "dlogits" in gpu:
        ref_dl = rr.dlogits
        got = gpu["dlogits"]
        num = np.linalg.norm(got - ref_dl)
        den = np.linalg.norm(ref_dl)
        errs["dlogits_rel_l2"] = float(num / den) if den > 0 else float(num)
        assert (errs["dlogits_rel_l2"] <= dl_rel) if den > 0 else num == 0.0, errs
        zero_rows = (rr.s == 0.0) & ~nb
        assert np.all(got[zero_rows] == 0.0), "rows with s = 0 must be exactly zero"
        # and row by row: every row with s != 0 within the same 1e-2 relative L2, so that a
        # single wrong row cannot hide in the batch norm.  A row whose target is nearly certain
        # (p_y -> 1) has an exact gradient s (p - onehot) of norm ~ |s| (1 - p_y), far below
        # what p_y - 1 resolves in fp32 (|s| 2^-24 per entry); such rows are measured against
        # the floor 2^-16 |s| (the per-row dlogits criterion).
        live = (rr.s != 0.0) & ~nb
        if live.any():
            rn = np.linalg.norm(got[live] - ref_dl[live], axis=1)
            rd = np.linalg.norm(ref_dl[live], axis=1)
            row_rel = rn / np.maximum(rd, 2.0 ** -16 * np.abs(rr.s[live]))
            errs["dlogits_row_rel_l2_max"] = float(np.max(row_rel))
            assert np.all(row_rel <= dl_rel), (int(np.argmax(row_rel)), errs["dlogits_row_rel_l2_max"])
        # padding columns [V, ld) are never written
        raw = gpu["dlogits_raw"]
        if raw.shape[1] > batch.V:
            pad = raw[:, batch.V:]
            expect = logits_pad if gpu["inplace"] else np.uint16(0x7FC3)
            assert np.all(pad == expect), "padding columns of dlogits were written"
    return errs


def run_gpu_vp(batch, logits_bits, device, world, chunks=1, grad_scale=1.0, eps=0.2,
               eps_hi=None, norm="seq", traj_mask=None, want_dlogits=True, calls=1,
               shard_cols=None, lag=0, dynamic_rows=0):
    """The vocabulary-parallel path (NEXT(3)) with all `world` ranks in one cooperative
    launch on one GPU: the logits are cut into world column shards of shard_cols columns,
    the per-rank dlogits shards are re-assembled into [T, ld] (padding left 0x7FC3).
    `calls` > 1 repeats the whole loss on the same exchange buffers (epoch counting)."""
    db = G.DeviceBatch.from_host(batch, device)
    mask_d = None if traj_mask is None else torch.from_numpy(
        np.ascontiguousarray(traj_mask, np.uint8)).to(device)
    loss = G.GrpoAsyncLoss(eps=eps, grad_scale=grad_scale, eps_hi=eps_hi, norm=norm,
                           traj_mask=mask_d)
    vo = loss.validate(db)
    adv, inv = loss.advantage(db)
    T, ld, V = batch.T, batch.ld, batch.V
    comm = G.VpGroup.local(world, V, T, device, shard_cols)
    comm.lag = lag
    comm.dynamic_rows = dynamic_rows
    sc = comm.shard_cols
    ld_s = sc  # shard row stride (a multiple of 8)
    full = np.full((T, sc * world), 0x7FC1, np.uint16)
    full[:, :V] = logits_bits[:, :V]
    shards = [to_dev_bits(np.ascontiguousarray(full[:, q * sc:(q + 1) * sc]), device)
              for q in range(world)]
    assert all(s.shape == (T, ld_s) for s in shards)
    bounds = np.linspace(0, T, chunks + 1).astype(np.int64)
    for _ in range(calls):
        dsh = [torch.full((T, ld_s), 0x7FC3, dtype=torch.int16, device=device)
               for _ in range(world)] if want_dlogits else None
        logp = torch.full((T,), float("nan"), device=device)
        lse = torch.full((T,), float("nan"), device=device)
        scale = torch.full((T,), float("nan"), device=device)
        traj_sum = torch.zeros(batch.N, dtype=torch.float64, device=device)
        stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=device)
        for c in range(chunks):
            b, e = int(bounds[c]), int(bounds[c + 1])
            loss.loss_chunk_vp(comm, [s[b:e] for s in shards], b, e - b, db.target_ids[b:e],
                               db.logp_behav[b:e], db.cu_seqlens, adv, inv, traj_sum, stats,
                               dshards=[d[b:e] for d in dsh] if dsh else None,
                               logp_out=logp[b:e], lse_out=lse[b:e], scale_out=scale[b:e], V=V)
        torch.cuda.synchronize()
    out = dict(
        traj_flags=vo.traj_flags.cpu().numpy().view(np.uint32)[:batch.N],
        group_count=vo.group_count.cpu().numpy(),
        stale_hist=vo.stale_hist.cpu().numpy().reshape(batch.P, batch.K + 1),
        summary=vo.summary_dict(),
        adv=adv.cpu().numpy(), inv_norm=inv.cpu().numpy(),
        logp=logp.cpu().numpy().astype(np.float64), lse=lse.cpu().numpy().astype(np.float64),
        scale=scale.cpu().numpy().astype(np.float64),
        traj_sum=traj_sum.cpu().numpy(), stats=stats.cpu().numpy(),
        launches=loss.launches, inplace=False, epoch=comm.epoch)
    if want_dlogits:
        cat = np.concatenate([d.cpu().numpy().view(np.uint16) for d in dsh], axis=1)
        raw = np.full((T, ld), 0x7FC3, np.uint16)
        raw[:, :V] = cat[:, :V]
        out["dlogits_raw"] = raw
        out["dlogits"] = bf16_bits_to_f32(raw[:, :V]).astype(np.float64)
        out["shard_pad_untouched"] = bool(np.all(cat[:, V:] == 0x7FC3))
    return out


def lmhead_accum_J_bound(batch, X_bits, W_bits, ref):
    """DESIGN.md Z25: on the LM-head path the logits z = X W^T are fp32 tensor-core sums, one
    accumulator rounding per tcgen05.mma K-step of 16 products, each within 1 ulp
    (<= 2^-23 |acc|) -- so |dz_tv| <= ceil(d/16) 2^-23 sum_k |x_tk| |w_vk|, |d logp_t| <=
    2 max_v |dz_tv|, and J (eq:grpo_async) moves by at most sum over unclipped tokens of
    inv_norm |A| r |d logp_t|.  A bound from the inputs alone (no GPU value enters it)."""
    X = np.abs(bf16_bits_to_f32(X_bits).astype(np.float64))
    W = np.abs(bf16_bits_to_f32(W_bits).astype(np.float64))
    d = X.shape[1]
    zabs = np.zeros(X.shape[0])
    for v0 in range(0, W.shape[0], 16384):
        zabs = np.maximum(zabs, (X @ W[v0:v0 + 16384].T).max(axis=1))
    B = 2.0 * -(-d // 16) * 2.0 ** -23 * zabs
    rr = ref["rows"]
    tok = np.repeat(np.arange(batch.N), batch.lengths)
    live = ~rr.clipped
    return float(np.sum((ref["inv_norm"][tok] * np.abs(ref["adv"][tok]) * rr.r * B)[live]))


def lmhead_batch(name, seed, d, sigma=0.05):
    """A synth batch with LM-head inputs X, W and behaviour log-probs built from the
    oracle's own logp (test-side input construction): logp_w = f32(logp - delta),
    delta ~ N(0, (sigma (1 + staleness gap))^2)."""
    import dataclasses

    from synth.gen import lmhead_inputs, make_batch
    b = make_batch(name, seed)
    X, W = lmhead_inputs(b.T, b.V, d, seed)
    z = O.lmhead_logits(X, W)
    m = z.max(axis=1, keepdims=True)
    lse = (m + np.log(np.exp(z - m).sum(axis=1, keepdims=True)))[:, 0]
    logp = z[np.arange(b.T), b.target_ids] - lse
    gap = np.repeat(b.v_theta - b.version_ids, b.lengths).astype(np.float64)
    rng = np.random.default_rng(seed + 77)
    lw = (logp - rng.normal(size=b.T) * sigma * (1 + gap)).astype(np.float32)
    return dataclasses.replace(b, logp_behav=lw), X, W


def run_gpu_lmhead(batch, X, W, device, chunks=1, want_grads=True, grad_scale=1.0, eps=0.2,
                   eps_hi=None, norm="seq", traj_mask=None):
    """NEXT(2) on the GPU: validate, advantage, lmhead_fwd over row chunks, lmhead_bwd."""
    db = G.DeviceBatch.from_host(batch, device)
    mask_d = None if traj_mask is None else torch.from_numpy(
        np.ascontiguousarray(traj_mask, np.uint8)).to(device)
    loss = G.GrpoAsyncLoss(eps=eps, grad_scale=grad_scale, eps_hi=eps_hi, norm=norm,
                           traj_mask=mask_d)
    vo = loss.validate(db)
    adv, inv = loss.advantage(db)
    T, V = batch.T, batch.V
    d = X.shape[1]
    Xd = to_dev_bits(X, device).view(torch.bfloat16)
    Wd = to_dev_bits(W, device).view(torch.bfloat16)
    logp = torch.full((T,), float("nan"), device=device)
    lse = torch.full((T,), float("nan"), device=device)
    scale = torch.full((T,), float("nan"), device=device)
    traj_sum = torch.zeros(batch.N, dtype=torch.float64, device=device)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=device)
    ld = (V + 7) // 8 * 8 + 8
    dz = torch.full((T, ld), 0x7FC3, dtype=torch.int16, device=device).view(torch.bfloat16)
    dX = torch.full((T, d), float("nan"), device=device).bfloat16()
    dW = torch.zeros((V, d), dtype=torch.float32, device=device)
    bounds = np.linspace(0, T, chunks + 1).astype(np.int64)
    for c in range(chunks):
        b, e = int(bounds[c]), int(bounds[c + 1])
        loss.lmhead_fwd(Xd[b:e], Wd, b, e - b, db.target_ids[b:e], db.logp_behav[b:e],
                        db.cu_seqlens, adv, inv, traj_sum, stats, logp_out=logp[b:e],
                        lse_out=lse[b:e], scale_out=scale[b:e])
        if want_grads:
            loss.lmhead_bwd(Xd[b:e], Wd, e - b, db.target_ids[b:e], lse[b:e], scale[b:e], dz[b:e],
                            dhidden=dX[b:e], dW=dW)
    torch.cuda.synchronize()
    out = dict(
        traj_flags=vo.traj_flags.cpu().numpy().view(np.uint32)[:batch.N],
        group_count=vo.group_count.cpu().numpy(),
        stale_hist=vo.stale_hist.cpu().numpy().reshape(batch.P, batch.K + 1),
        summary=vo.summary_dict(), adv=adv.cpu().numpy(), inv_norm=inv.cpu().numpy(),
        logp=logp.cpu().numpy().astype(np.float64), lse=lse.cpu().numpy().astype(np.float64),
        scale=scale.cpu().numpy().astype(np.float64), traj_sum=traj_sum.cpu().numpy(),
        stats=stats.cpu().numpy(), launches=loss.launches, inplace=False)
    if want_grads:
        raw = dz.view(torch.int16).cpu().numpy().view(np.uint16)
        out["dlogits_raw"] = raw
        out["dlogits"] = bf16_bits_to_f32(raw[:, :V]).astype(np.float64)
        out["dz_pad_untouched"] = bool(np.all(raw[:, V:] == 0x7FC3))
        out["dhidden"] = dX.float().cpu().numpy().astype(np.float64)
        out["dW"] = dW.cpu().numpy().astype(np.float64)
    return out
