"""NEXT(2) x NEXT(3): the tensor-parallel LM head fused with the loss on R GPUs (torchrun).

Every rank holds the hidden states of the chunk and W rows [q*Vs, (q+1)*Vs); the forward
all-gathers the per-row softmax partials (16 B per row and rank) over NCCL, the backward
all-reduces the dhidden partials.  Part 1: parity against the fp64 oracle on a small case.
Part 2: timing on the LM-head bench workload (R = 8190 rows, d = 5120, V = 152064), max over
ranks, against the single-GPU fused LM head.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/lmhead_tp.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_26256_b200 as G  # noqa: E402
from synth.gen import make_batch  # noqa: E402


from paper_2604_26256_b200 import _lib as L_  # noqa: E402

TIMERS = [torch.cuda.Event(enable_timing=True) for _ in range(6)]


class FusedDX:
    """Slot buffers for grpo_async_lmhead_tp_dx in torch symmetric memory (peer pointers)."""

    def __init__(self, n, d, world, dev):
        import torch.distributed._symmetric_memory as symm
        self.rpr = -(-n // world)
        # two halves: call e writes half e % 2 (include/grpo_async.h, grpo_async_lmhead_tp_dx)
        self.buf = symm.empty(2 * world * self.rpr * d, dtype=torch.float32, device=dev)
        self.h = symm.rendezvous(self.buf, dist.group.WORLD)
        self.ptrs = [self.h.get_buffer(q, (2 * world * self.rpr * d,), torch.float32).data_ptr()
                     for q in range(world)]
        self.flag = torch.zeros(1, device=dev)
        self.epoch = 0


def run(loss, db, X, W, V, R0, n, rank, world, lw=None, overlap=False, fused=None):
    d = X.shape[1]
    Vs = -(-V // world)
    off = rank * Vs
    Wq = W[off:min(off + Vs, V)].contiguous() if W.shape[0] == V else W
    T = n
    logp = torch.empty(T, device=X.device)
    lse = torch.empty(T, device=X.device)
    scale = torch.empty(T, device=X.device)
    ts = torch.zeros(db.N, dtype=torch.float64, device=X.device)
    st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=X.device)
    adv, inv = loss.advantage(db)
    lwx = db.logp_behav[R0:R0 + n] if lw is None else lw
    loss.lmhead_tp_fwd(X, Wq, off, V, R0, n, db.target_ids[R0:R0 + n], lwx, db.cu_seqlens, adv,
                       inv, ts, st, logp_out=logp, lse_out=lse, scale_out=scale)
    Vq = Wq.shape[0]
    dz = torch.empty((n, (Vq + 7) // 8 * 8), dtype=torch.bfloat16, device=X.device)
    dX = torch.empty((n, d), dtype=torch.float32, device=X.device)
    dW = torch.zeros((Vq, d), dtype=torch.float32, device=X.device)
    if fused is not None:  # one GEMM -> reduce-scatter kernel over peer memory, then dW
        from paper_2604_26256_b200 import _lib as L
        tm = TIMERS
        tm[0].record()
        loss.lmhead_tp_bwd(X, Wq, off, n, db.target_ids[R0:R0 + n], lse, scale, dz)
        tm[1].record()
        L.grpo_async_lmhead_tp_dx(dz, dz.shape[1], Wq, n, d, Vq, world, rank, fused.ptrs, fused.epoch)
        tm[2].record()
        L.grpo_async_lmhead_dw(X, n, d, Vq, dz, dz.shape[1], dW)
        tm[3].record()
        # every rank's tiles have landed in their owners' slots: a 1-element all-reduce is
        # stream-ordered after the GEMM (dist.barrier() would synchronize the host)
        dist.all_reduce(fused.flag)
        tm[4].record()
        rows = max(0, min(fused.rpr, n - rank * fused.rpr))
        mine = torch.empty((max(rows, 1), d), dtype=torch.float32, device=X.device)
        L.grpo_async_lmhead_tp_dx_reduce(fused.buf, world, n, d, rank, mine, fused.epoch)
        fused.epoch += 1
        tm[5].record()
        return logp, st, mine[:rows], dW, dz
    if overlap:  # the dhidden all-reduce overlaps the dW GEMM
        h = loss.lmhead_tp_bwd(X, Wq, off, n, db.target_ids[R0:R0 + n], lse, scale, dz,
                               dhidden_partial=dX, dW_shard=dW,
                               allreduce_async=lambda t: dist.all_reduce(t, async_op=True))
        h.wait()
    else:
        loss.lmhead_tp_bwd(X, Wq, off, n, db.target_ids[R0:R0 + n], lse, scale, dz,
                           dhidden_partial=dX, dW_shard=dW)
        dist.all_reduce(dX)
    return logp, st, dX, dW, dz


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    out = {"world": world}
    # ---- parity (small): oracle on the whole W on every rank
    import oracle.oracle as O
    from tests.gpu_util import lmhead_batch, to_dev_bits
    b, Xb, Wb = lmhead_batch("ragged", 7, 128)
    ref = O.run_batch_lmhead(b, Xb, Wb, std_floor=float(np.float32(1e-8)))
    db = G.DeviceBatch.from_host(b, dev)
    X = to_dev_bits(Xb, dev).view(torch.bfloat16)
    W = to_dev_bits(Wb, dev).view(torch.bfloat16)
    logp, st, dX, dW, dz = run(G.GrpoAsyncLoss(), db, X, W, b.V, 0, b.T, rank, world)
    torch.cuda.synchronize(dev)
    err = {"logp_max_abs": float(np.max(np.abs(logp.cpu().numpy() - ref["rows"].logp))),
           "J_gpu": float(st[G.STAT_J].item()), "J_ref": float(ref["J"]),
           "dX_rel_l2": float(np.linalg.norm(dX.cpu().numpy() - ref["dhidden"]) / np.linalg.norm(ref["dhidden"]))}
    ok = err["logp_max_abs"] <= 2e-3 and err["dX_rel_l2"] <= 1e-2 and \
        abs(err["J_gpu"] - err["J_ref"]) <= 1e-5 * max(abs(err["J_ref"]), 1e-3)
    okt = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    out["parity_rank0"] = err
    out["parity_all_ranks_ok"] = bool(okt.item())
    # ---- timing on the LM-head bench workload
    bb = make_batch("prod", 0, period=8192)
    n = int(bb.cu_seqlens[int(np.searchsorted(bb.cu_seqlens, 8192, side="right") - 1)])
    V, d = bb.V, 5120
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    Xt = torch.randn((n, d), device=dev, generator=g).bfloat16()
    Wt = (torch.randn((V, d), device=dev, generator=g) * (2.5 / d ** 0.5)).bfloat16()
    Vs = -(-V // world)
    Wq = Wt[rank * Vs:min((rank + 1) * Vs, V)].contiguous()
    del Wt
    dbb = G.DeviceBatch.from_host(bb, dev)
    loss = G.GrpoAsyncLoss()

    fused = FusedDX(n, d, world, dev)
    # the fused dhidden (this rank's rows) against the NCCL all-reduce path
    _, _, dx_ref, _, _ = run(loss, dbb, Xt, Wq, V, 0, n, rank, world)
    _, _, dx_f, _, _ = run(loss, dbb, Xt, Wq, V, 0, n, rank, world, fused=fused)
    r0 = rank * fused.rpr
    rel = (torch.linalg.norm(dx_f - dx_ref[r0:r0 + dx_f.shape[0]]) /
           torch.linalg.norm(dx_ref[r0:r0 + dx_f.shape[0]])).reshape(1)
    dist.all_reduce(rel, op=dist.ReduceOp.MAX)
    out["fused_dx_vs_nccl_rel_l2"] = float(rel.item())

    def timed(overlap, fz=None):
        for _ in range(2):
            run(loss, dbb, Xt, Wq, V, 0, n, rank, world, overlap=overlap, fused=fz)
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run(loss, dbb, Xt, Wq, V, 0, n, rank, world, overlap=overlap, fused=fz)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = torch.tensor([e0.elapsed_time(e1) / 5], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    ms = timed(False)
    ms_ovl = timed(True)
    ms_fused = timed(False, fused)
    torch.cuda.synchronize(dev)
    out["ms_fused_path_parts"] = {"dz": TIMERS[0].elapsed_time(TIMERS[1]),
                                  "dx_gemm_reduce_scatter": TIMERS[1].elapsed_time(TIMERS[2]),
                                  "dW_gemm": TIMERS[2].elapsed_time(TIMERS[3]),
                                  "flag_allreduce": TIMERS[3].elapsed_time(TIMERS[4]),
                                  "slot_sum": TIMERS[4].elapsed_time(TIMERS[5])}
    out["timing"] = {"rows": n, "d": d, "V": V, "shard_cols": Vs, "ms_fwd_bwd_step": ms,
                     "ms_fwd_bwd_step_allreduce_overlap_dw": ms_ovl,
                     "ms_fwd_bwd_step_fused_dx_reduce_scatter": ms_fused,
                     "tflops_per_gpu": 8.0 * n * Vs * d / ms / 1e9}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
