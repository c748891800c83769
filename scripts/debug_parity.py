"""Ad-hoc diagnostics for parity failures (prints, never asserts)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from tests.test_gpu_parity import _adversarial_batch, _case, KERNELS
from tests.gpu_util import run_gpu, run_oracle, to_dev_bits
import paper_2604_26256_b200 as G

dev = torch.device("cuda:0")
np.set_printoptions(linewidth=200, precision=6)
# 1. adversarial NaN
V = 4099
rng = np.random.default_rng(1)
rows = []
rows.append((np.zeros(V), 0)); rows.append((np.zeros(V), V - 1))
z = rng.normal(size=V); z[17] = 60.0; rows.append((z, 17))
z = rng.normal(size=V); z[17] = 60.0; rows.append((z, 5))
z = rng.normal(size=V); z[::3] = -np.inf; rows.append((z, 1))
z = rng.normal(size=V) * 30; rows.append((z, 100))
z = rng.normal(size=V) + 1e4; rows.append((z, 7))
z = np.full(V, -1e30); z[V - 2] = 0.0; rows.append((z, V - 2))
for _ in range(8):
    rows.append((rng.normal(size=V) * 3, int(rng.integers(0, V))))
b, bits = _adversarial_batch(V, rows)
ref = run_oracle(b, bits)
for tune in KERNELS:
    gpu = run_gpu(b, bits, dev, tune=tune)
    print("tune", tune)
    print(" ref logp", ref["rows"].logp)
    print(" gpu logp", gpu["logp"])
    print(" ref lse ", ref["rows"].lse)
    print(" gpu lse ", gpu["lse"])
    print(" lw", b.logp_behav)
# 2. fused vs unfused bwd
b, bits = _case("mid152k", 5)
gpu = run_gpu(b, bits, dev)
lg = to_dev_bits(bits, dev)
out = torch.full_like(lg, 0x7FC3)
G.grpo_async_loss_bwd(lg, b.T, b.V, b.ld, torch.from_numpy(b.target_ids).to(dev),
                      torch.from_numpy(gpu["lse"].astype(np.float32)).to(dev),
                      torch.from_numpy(gpu["scale"].astype(np.float32)).to(dev), 1.0, out)
torch.cuda.synchronize()
o = out.cpu().numpy().view(np.uint16)
f = gpu["dlogits_raw"]
bad = np.argwhere(o != f)
print("bwd mismatches", len(bad), "of", o.size)
for r, c in bad[:20]:
    print(r, c, hex(o[r, c]), hex(f[r, c]), "target", b.target_ids[r], "scale", gpu["scale"][r], "V", b.V)
