"""NEXT(2) measurement: the LM-head-fused loss on one B200.

Workload: one chunk of --rows response tokens of the prod batch,
hidden size d = 5120 and V = 152064 (Qwen2.5-32B, the paper's dense model),
bf16 hidden states X ~ N(0,1) and LM-head weight W ~ N(0, (2.5/sqrt d)^2) generated on
the device; behaviour log-probs = the model's own logp minus N(0, (0.03 (1+gap))^2)
(what a rollout engine records), set once before timing.

Timed with CUDA events on the launching stream after warm-up (max of nothing: one GPU):
  fwd   grpo_async_lmhead_fwd   (tcgen05 GEMM + loss epilogue; logits never stored)
  bwd   grpo_async_lmhead_bwd   (tcgen05 GEMM recompute + dz epilogue; tcgen05 dX, dW GEMMs)
  the GEMMs alone: grpo_async_lmhead_dx (dX = dz W) and grpo_async_lmhead_dw (dW += dz^T X)
  unfused on the same data, every kernel ours: grpo_async_lmhead_logits (tcgen05, bf16
  logits) -> grpo_async_loss_fwd (dlogits) -> grpo_async_lmhead_dx -> grpo_async_lmhead_dw;
  and the same with torch.matmul (cuBLAS) GEMMs, as a library baseline.
Prints one JSON line.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_26256_b200 as G  # noqa: E402
from paper_2604_26256_b200 import _lib as L  # noqa: E402
from synth.gen import make_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--d", type=int, default=5120)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--skip-unfused", action="store_true")
    ap.add_argument("--cta-group", type=int, default=2, help="1 or 2 (tcgen05 cta_group::2 pairs)")
    args = ap.parse_args()
    L.grpo_async_lmhead_set_cta_group(args.cta_group)
    dev = torch.device("cuda", 0)
    b = make_batch("prod", 0, period=args.rows)
    R, V, d = min(args.rows, b.T), b.V, args.d
    # whole trajectories only: cut the batch at a trajectory boundary <= R
    n_traj = int(np.searchsorted(b.cu_seqlens, R, side="right") - 1)
    R = int(b.cu_seqlens[n_traj])
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    X = torch.randn((R, d), device=dev, generator=g).bfloat16()
    W = (torch.randn((V, d), device=dev, generator=g) * (2.5 / d ** 0.5)).bfloat16()
    tgt = db.target_ids[:R]
    logp = torch.empty(R, device=dev)
    lse = torch.empty(R, device=dev)
    scale = torch.empty(R, device=dev)
    ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
    st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    lw0 = db.logp_behav[:R].clone()
    loss.lmhead_fwd(X, W, 0, R, tgt, lw0, db.cu_seqlens, adv, inv, ts, st, logp_out=logp)
    gap = torch.from_numpy(np.repeat(b.v_theta - b.version_ids, b.lengths)[:R]).to(dev).float()
    lw = (logp - torch.randn(R, device=dev, generator=g) * 0.03 * (1 + gap)).float().contiguous()
    ld = (V + 7) // 8 * 8
    dz = torch.empty((R, ld), dtype=torch.bfloat16, device=dev)
    dX = torch.empty((R, d), dtype=torch.bfloat16, device=dev)
    dW = torch.zeros((V, d), dtype=torch.float32, device=dev)

    def fwd():
        ts.zero_()
        st.zero_()
        loss.lmhead_fwd(X, W, 0, R, tgt, lw, db.cu_seqlens, adv, inv, ts, st, logp_out=logp,
                        lse_out=lse, scale_out=scale)

    def bwd():
        loss.lmhead_bwd(X, W, R, tgt, lse, scale, dz, dhidden=dX, dW=dW)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    # kernel-only time of the tcgen05 launches via the library's event tracing
    def traced(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        L.grpo_profile_enable(True)
        L.grpo_profile_collect()
        for _ in range(args.steps):
            fn()
        n, tot = L.grpo_profile_collect()
        L.grpo_profile_enable(False)
        return tot / max(n, 1)

    ms_fwd = timed(fwd)
    plan_fwd = G.grpo_async_last_plan()
    ms_fwd_kernel = traced(fwd)
    ms_bwd = timed(bwd)
    fl = 2.0 * R * V * d
    out = {"workload": f"lmhead prod chunk R={R} d={d} V={V}", "rows": R, "d": d, "V": V,
           "cta_group": args.cta_group,
           "ms_fwd": ms_fwd, "ms_fwd_tcgen05_kernel": ms_fwd_kernel, "ms_bwd": ms_bwd,
           "fwd_tflops": fl / ms_fwd / 1e9, "fwd_kernel_tflops": fl / ms_fwd_kernel / 1e9,
           "bwd_tflops": 3 * fl / ms_bwd / 1e9, "plan_fwd": plan_fwd,
           "J": float(st[G.STAT_J].item()),
           "clipped_frac": float(st[G.STAT_CLIPPED].item()) / R}
    # the dz kernel alone (bwd without the dX / dW GEMMs), then each GEMM alone on that dz
    out["ms_dz_kernel"] = timed(lambda: loss.lmhead_bwd(X, W, R, tgt, lse, scale, dz))
    out["dz_kernel_tflops"] = fl / out["ms_dz_kernel"] / 1e9
    out["ms_dx_gemm"] = timed(lambda: L.grpo_async_lmhead_dx(dz, ld, W, R, d, V, dX))
    out["dx_gemm_tflops"] = fl / out["ms_dx_gemm"] / 1e9
    out["ms_dw_gemm"] = timed(lambda: L.grpo_async_lmhead_dw(X, R, d, V, dz, ld, dW))
    out["dw_gemm_tflops"] = fl / out["ms_dw_gemm"] / 1e9
    out["ms_fused_fwd_bwd"] = ms_fwd + ms_bwd
    if not args.skip_unfused:
        lg = torch.empty((R, ld), dtype=torch.bfloat16, device=dev)
        dl = torch.empty((R, ld), dtype=torch.bfloat16, device=dev)

        def unfused_ours():
            L.grpo_async_lmhead_logits(X, W, R, d, V, lg, ld)
            ts.zero_()
            st.zero_()
            loss.loss_chunk(lg, 0, R, tgt, lw, db.cu_seqlens, adv, inv, ts, st, dlogits=dl, V=V)
            L.grpo_async_lmhead_dx(dl, ld, W, R, d, V, dX)
            L.grpo_async_lmhead_dw(X, R, d, V, dl, ld, dW)

        out["ms_unfused_fwd_bwd"] = timed(unfused_ours)
        out["ms_logits_gemm"] = timed(lambda: L.grpo_async_lmhead_logits(X, W, R, d, V, lg, ld))
        dWb = torch.empty((V, d), dtype=torch.bfloat16, device=dev)

        def unfused_cublas():
            torch.matmul(X, W.t(), out=lg[:, :V]) if ld == V else lg[:, :V].copy_(X @ W.t())
            ts.zero_()
            st.zero_()
            loss.loss_chunk(lg, 0, R, tgt, lw, db.cu_seqlens, adv, inv, ts, st, dlogits=dl, V=V)
            torch.matmul(dl[:, :V], W, out=dX)
            torch.matmul(dl[:, :V].t(), X, out=dWb)  # (bf16 out, the same GEMM work)

        out["ms_unfused_fwd_bwd_torch_cublas"] = timed(unfused_cublas)
        del lg, dl
    out["tensor_peak_tflops"] = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
