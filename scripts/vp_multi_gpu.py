"""NEXT(3) on R GPUs: the vocabulary-parallel fused loss (grpo_async_loss_fwd_vp) with
each rank holding one column shard of the logits and exchanging its per-row partial
over NVLink peer memory (torch symmetric memory mappings).

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/vp_multi_gpu.py

Part 1 (parity): mid152k seed 5 -- every rank checks the per-row outputs and its own
dlogits columns against the fp64 oracle (test infrastructure, as in tests/).
Part 2 (timing): a prod chunk of --rows rows, each rank reads rows x V/R logits and
writes the same dlogits; CUDA-event time of the vp kernel call, max over ranks,
against the single-GPU fused kernel on the unsharded chunk (rank 0).
Prints one JSON line on rank 0.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_26256_b200 as G  # noqa: E402
from synth import gpu as SG  # noqa: E402
from synth.gen import bf16_bits_to_f32, make_batch  # noqa: E402


def parity(rank, world, dev):
    import oracle.oracle as O
    b = make_batch("mid152k", 5)
    bits = b.logits_bits()
    ref = O.run_batch(b, bits, eps=0.2, grad_scale=1.0, std_floor=float(np.float32(1e-8)),
                      want_dlogits=True)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    loss.validate(db)
    adv, inv = loss.advantage(db)
    T, V = b.T, b.V
    comm = G.VpGroup.from_symmetric(V, T, dev)
    sc = comm.shard_cols
    full = np.full((T, sc * world), 0x7FC1, np.uint16)
    full[:, :V] = bits[:, :V]
    mine = torch.from_numpy(np.ascontiguousarray(full[:, rank * sc:(rank + 1) * sc]).view(np.int16)).to(dev)
    dmine = torch.full_like(mine, 0x7FC3)
    logp = torch.full((T,), float("nan"), device=dev)
    scale = torch.full((T,), float("nan"), device=dev)
    traj_sum = torch.zeros(b.N, dtype=torch.float64, device=dev)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    loss.loss_chunk_vp(comm, [mine], 0, T, db.target_ids, db.logp_behav, db.cu_seqlens, adv, inv,
                       traj_sum, stats, dshards=[dmine], logp_out=logp, scale_out=scale, V=V)
    torch.cuda.synchronize(dev)
    rr = ref["rows"]
    lo, hi = rank * sc, min((rank + 1) * sc, V)
    got = bf16_bits_to_f32(dmine.cpu().numpy().view(np.uint16)[:, :hi - lo]).astype(np.float64)
    want = rr.dlogits[:, lo:hi]
    res = dict(
        logp_max_abs=float(np.max(np.abs(logp.cpu().numpy() - rr.logp))),
        J_gpu=float(stats[G.STAT_J].item()), J_ref=float(ref["J"]),
        dlogits_rel_l2=float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)),
        pad_untouched=bool(np.all(dmine.cpu().numpy().view(np.uint16)[:, hi - lo:] == 0x7FC3)))
    res["ok"] = (res["logp_max_abs"] <= 2e-3 and res["dlogits_rel_l2"] <= 1e-2 and
                 abs(res["J_gpu"] - res["J_ref"]) <= 1e-5 * max(abs(res["J_ref"]), 1e-2) and
                 res["pad_untouched"])
    return res


def timing(rank, world, dev, rows, steps, warmup):
    b = make_batch("prod", 0, period=rows)
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    V = b.V
    R = min(rows, b.T)
    comm = G.VpGroup.from_symmetric(V, R, dev)
    sc = comm.shard_cols
    full = torch.empty((R, b.ld), dtype=torch.int16, device=dev)
    spec = b.logits
    spec.period = rows
    SG.fill_logits(full, spec, 0, R, V)
    lo, hi = rank * sc, min((rank + 1) * sc, V)
    mine = torch.full((R, sc), 0x7FC1, dtype=torch.int16, device=dev)
    mine[:, :hi - lo] = full[:, lo:hi]
    dmine = torch.empty_like(mine)
    traj_sum = torch.zeros(b.N, dtype=torch.float64, device=dev)
    stats = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    tgt, lw = db.target_ids[:R], db.logp_behav[:R]

    logp_chk = torch.empty(R, device=dev)

    def vp(logp_out=None):
        loss.loss_chunk_vp(comm, [mine], 0, R, tgt, lw, db.cu_seqlens, adv, inv, traj_sum, stats,
                           dshards=[dmine], V=V, logp_out=logp_out)

    # the exchange protocol must give the same bits on the first call and after hundreds of
    # calls on the same buffers (epoch parity, tags), in every schedule
    vp(logp_chk)
    torch.cuda.synchronize(dev)
    first = logp_chk.clone()
    d_first = dmine.clone()

    def timed(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    modes = {}
    for name, lag, dyn in (("static_lag0", 0, 0), ("static_lag1", 1, 0), ("dynamic_lag0", 0, 1),
                           ("dynamic_lag1", 1, 1), ("ring_delay1", 2, 0), ("ring_delay2", 3, 0),
                           ("ring_delay3", 4, 0)):
        comm.lag, comm.dynamic_rows = lag, dyn
        modes[name] = timed(vp)
    comm.lag, comm.dynamic_rows = 0, 0
    ms_vp = timed(vp)
    plan = G.grpo_async_last_plan()
    vp(logp_chk)
    torch.cuda.synchronize(dev)
    same = bool(torch.equal(first, logp_chk) and torch.equal(d_first, dmine))
    ok = torch.tensor([1 if same else 0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # the same per-rank bytes through the single-GPU kernel: a V = shard_cols problem
    tgt_h = tgt % sc

    def single_half():
        loss.loss_chunk(mine, 0, R, tgt_h, lw, db.cu_seqlens, adv, inv, traj_sum, stats,
                        dlogits=dmine, V=sc)
    ms_half = timed(single_half)
    del mine, dmine
    ms_single = None
    if rank == 0:
        dfull = torch.empty_like(full)

        def single():
            loss.loss_chunk(full, 0, R, tgt, lw, db.cu_seqlens, adv, inv, traj_sum, stats,
                            dlogits=dfull, V=V)
        for _ in range(warmup):
            single()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            single()
        e1.record()
        torch.cuda.synchronize(dev)
        ms_single = e0.elapsed_time(e1) / steps
    dist.barrier()
    bytes_rank = R * (hi - lo) * 2 * 2
    return dict(rows=R, V=V, shard_cols=sc, ms_vp_step=ms_vp, ms_vp_modes=modes,
                bitwise_stable_after_epochs=bool(ok.item()), epochs=comm.epoch,
                ms_single_kernel_on_shard=ms_half,
                ms_single_gpu=ms_single,
                vp_GBps_per_rank=bytes_rank / ms_vp / 1e6,
                speedup_vs_single=(ms_single / ms_vp) if ms_single else None, plan=plan)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--skip-parity", action="store_true")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    out = {"world": world}
    if not args.skip_parity:
        p = parity(rank, world, dev)
        flags = torch.tensor([1 if p["ok"] else 0], device=dev)
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        out["parity_rank0"] = p
        out["parity_all_ranks_ok"] = bool(flags.item())
    out["timing"] = timing(rank, world, dev, args.rows, args.steps, args.warmup)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
