"""Small runs of every shipped kernel, for compute-sanitizer (one tool per invocation):

    compute-sanitizer --tool memcheck  python scripts/sanitize_case.py
    compute-sanitizer --tool racecheck python scripts/sanitize_case.py
    compute-sanitizer --tool synccheck python scripts/sanitize_case.py

Covers validate, advantage (+ sharded-rewards kernels), row info, the row-wise kernel K3b
(single CTA and 2-CTA cluster), the ring kernel K3c (16 KB / 32 KB slots = the production
stream_kernel<512,1,2048,1>, two CTAs per SM, and the two-SM split-row cluster
stream_kernel<512,1,2048,2>), the segmented reductions, the unfused backward, the
vocabulary-parallel kernels (row-wise vp_kernel and the ring vp_stream_kernel, ranks
emulated on one GPU), and the LM-head tcgen05 kernels (forward stats, dz, logits, dX/dW
GEMMs, the tensor-parallel dX GEMM -> slot stores and its reduce)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_26256_b200 as G  # noqa: E402
from paper_2604_26256_b200 import _lib as L  # noqa: E402
from synth.gen import make_batch  # noqa: E402
from tests.gpu_util import lmhead_batch, run_gpu, run_gpu_lmhead, run_gpu_vp, to_dev_bits  # noqa: E402
from tests.test_gpu_parity import _adversarial_batch  # noqa: E402

dev = torch.device("cuda:0")
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "loss"):
    for name in ("tiny", "ragged"):
        b = make_batch(name, 0)
        bits = b.logits_bits()
        tunes = [None, {"kernel": 2}, {"kernel": 2, "cluster_size": 2, "ctas_per_sm": 2},
                 {"kernel": 3}, {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3},
                 {"kernel": 3, "chunk_kb": 16, "stages": 6, "lag": 3, "row_cache": 2, "ctas_per_sm": 256}]
        if b.V >= 16384:
            tunes.append({"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3, "cluster_size": 2})
        for tune in tunes:
            run_gpu(b, bits, dev, tune=tune, chunks=2)
        out = run_gpu(b, bits, dev, eps_hi=0.28, norm="token",
                      traj_mask=(np.arange(b.N) % 3 != 0).astype(np.uint8))
        lg = torch.from_numpy(bits.view(np.int16)).to(dev)
        dl = torch.empty_like(lg)
        G.grpo_async_loss_bwd(lg, b.T, b.V, b.ld, torch.from_numpy(b.target_ids).to(dev),
                              torch.from_numpy(out["lse"].astype(np.float32)).to(dev),
                              torch.from_numpy(out["scale"].astype(np.float32)).to(dev), 1.0, dl)
    print("loss kernels done", flush=True)
if which in ("all", "vp"):
    rng = np.random.default_rng(5)
    for V, world in ((4099, 2), (152064, 2)):  # row-wise vp_kernel; ring vp_stream_kernel
        rows = [(rng.normal(size=V), int(rng.integers(0, V))) for _ in range(12)]
        b, bits = _adversarial_batch(V, rows)
        run_gpu_vp(b, bits, dev, world, calls=2)
        run_gpu_vp(b, bits, dev, world, lag=1)
    print("vocabulary-parallel kernels done", flush=True)
if which in ("all", "lmhead"):
    b, X, W = lmhead_batch("tiny", 0, 128)
    for cg in (2, 1):
        L.grpo_async_lmhead_set_cta_group(cg)
        run_gpu_lmhead(b, X, W, dev)
    L.grpo_async_lmhead_set_cta_group(2)
    # tensor-parallel dX GEMM -> slot stores -> rank-order reduce, 2 ranks emulated
    T, V, d, R = b.T, b.V, 128, 2
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
    Vs, rpr = -(-V // R), -(-T // R)
    bufs = [torch.zeros((2, R, rpr, d), device=dev) for _ in range(R)]
    for q in range(R):
        Wq = Wd[q * Vs:min((q + 1) * Vs, V)].contiguous()
        ld = (Wq.shape[0] + 7) // 8 * 8
        dz = torch.zeros((T, ld), dtype=torch.bfloat16, device=dev)
        loss.lmhead_tp_bwd(Xd, Wq, q * Vs, T, db.target_ids, lse, scale, dz)
        L.grpo_async_lmhead_tp_dx(dz, ld, Wq, T, d, Wq.shape[0], R, q, bufs, 1)
    for q in range(R):
        o = torch.empty((rpr, d), device=dev)
        L.grpo_async_lmhead_tp_dx_reduce(bufs[q], R, T, d, q, o, 1)
    print("LM-head kernels done", flush=True)
torch.cuda.synchronize()
print("sanitize case done")
