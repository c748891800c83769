"""Small run of every kernel for compute-sanitizer (one tool per invocation)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from synth.gen import make_batch
from tests.gpu_util import run_gpu
import paper_2604_26256_b200 as G

dev = torch.device("cuda:0")
for name in ("tiny", "ragged"):
    b = make_batch(name, 0)
    bits = b.logits_bits()
    for tune in ({"kernel": 1}, {"kernel": 2}, {"kernel": 2, "cluster_size": 2, "ctas_per_sm": 2},
                 {"kernel": 1, "cluster_size": 4}):
        out = run_gpu(b, bits, dev, tune=tune)
    out = run_gpu(b, bits, dev, eps_hi=0.28, norm="token",
                  traj_mask=(np.arange(b.N) % 3 != 0).astype(np.uint8))
    lg = torch.from_numpy(bits.view(np.int16)).to(dev)
    dl = torch.empty_like(lg)
    G.grpo_async_loss_bwd(lg, b.T, b.V, b.ld, torch.from_numpy(b.target_ids).to(dev),
                          torch.from_numpy(out["lse"].astype(np.float32)).to(dev),
                          torch.from_numpy(out["scale"].astype(np.float32)).to(dev), 1.0, dl)
torch.cuda.synchronize()
print("sanitize case done")
