"""Write the full-batch golden values of a benchmark configuration with the oracle only.

    python scripts/make_golden_full.py prod 0 131072

Every one of the T rows goes through oracle_rows (fp64 two-pass log-softmax, ratio,
clip, min); logits come from synth/gen.py (logical row t = physical row t % period,
the benchmark's resident-chunk recipe).  Output: tests/golden/<config>_seed<s>_R<period>.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle.oracle as O  # noqa: E402
from synth.gen import make_batch  # noqa: E402

name, seed, period = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
b = make_batch(name, seed, period=period)
adv, inv, gc = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P, float(np.float32(1e-8)))
T = b.T
term = np.zeros(T)
r = np.zeros(T)
logp = np.zeros(T)
clipped = np.zeros(T, bool)
blk = 1024
t0 = time.time()
for p0 in range(0, period, blk):
    p1 = min(period, p0 + blk)
    phys = np.arange(p0, p1)
    bits = b.logits.rows_bits(phys)                  # physical rows p0..p1
    pad = np.zeros((len(phys), b.ld), np.uint16)
    pad[:, :b.V] = bits
    for rep in range(0, (T + period - 1) // period):
        rows = phys + rep * period
        sel = rows < T
        if not sel.any():
            continue
        rows = rows[sel]
        rr = O.rows(rows, pad[sel], b.V, b.target_ids[rows], b.logp_behav[rows], b.cu_seqlens,
                    adv, inv, 0.2, 1.0, want_dlogits=False)
        term[rows], r[rows], logp[rows], clipped[rows] = rr.term, rr.r, rr.logp, rr.clipped
    if p0 % (16 * blk) == 0:
        print(f"{p1}/{period} physical rows, {time.time() - t0:.0f} s", flush=True)
J, traj_sum = O.objective_tokens(b.cu_seqlens, inv, term)
tok_inv = np.repeat(inv, b.lengths)
near = int(((np.abs(r - (1 + np.float32(0.2))) <= 1e-5) | (np.abs(r - (1 - np.float32(0.2))) <= 1e-5)).sum())
out = {"_source": f"scripts/make_golden_full.py {name} {seed} {period} (oracle only; synth/gen.py inputs)",
       "config": name, "seed": seed, "period": period, "T": T, "N": b.N, "V": b.V,
       "J": J, "S_abs": float(np.sum(tok_inv * np.abs(term))), "n_clipped": int(clipped.sum()),
       "n_near_boundary": near, "sum_logp": float(logp.sum()),
       "traj_sum": traj_sum.tolist(), "seconds": time.time() - t0}
path = os.path.join(ROOT, "tests", "golden", f"{name}_seed{seed}_R{period}.json")
with open(path, "w") as f:
    json.dump(out, f)
print("wrote", path, "J", J, "seconds", time.time() - t0)
