"""Probe: the large-vocabulary row split two ways on ONE GPU -- K3c's two-SM cluster rows (DSMEM
exchange) against the vocabulary-parallel kernels with both column halves in one cooperative
launch (n_local = 2: the exchange through global memory; lag 0 = look-ahead ring, lag 2 =
pass 2 delayed by a row).  CUDA events, median of reps, fraction of the measured copy
bandwidth (4V + 29 B per row).  python scripts/probes/split_vs_vp.py [V] [rows]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import dataclasses  # noqa: E402

import paper_2604_26256_b200 as G  # noqa: E402
import synth.gpu as SG  # noqa: E402
from synth.gen import CONFIGS, make_batch  # noqa: E402

V = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
R = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
dev = torch.device("cuda:0")
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
cfg = dataclasses.replace(CONFIGS["large"], V=V)
b = make_batch(cfg, 0, period=R)
ld = b.ld
lg = torch.empty((R, ld), dtype=torch.int16, device=dev)
SG.fill_logits(lg, b.logits, 0, R, V)
dl = torch.empty_like(lg)
db = G.DeviceBatch.from_host(b, dev)
loss = G.GrpoAsyncLoss()
adv, inv = loss.advantage(db)
ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
comm = G.VpGroup.local(2, V, R, dev)
sc = comm.shard_cols
sh = [lg[:, :sc].contiguous(), torch.zeros((R, sc), dtype=torch.int16, device=dev)]
sh[1][:, :V - sc] = lg[:, sc:V]
dsh = [torch.empty((R, sc), dtype=torch.int16, device=dev) for _ in range(2)]


def k3c():
    loss.loss_chunk(lg, 0, R, db.target_ids[:R], db.logp_behav[:R], db.cu_seqlens, adv, inv, ts, st,
                    dlogits=dl, V=V)


def vp(lag):
    def f():
        comm.lag = lag
        loss.loss_chunk_vp(comm, sh, 0, R, db.target_ids[:R], db.logp_behav[:R], db.cu_seqlens, adv,
                           inv, ts, st, dshards=dsh, V=V)
    return f


cases = {"k3c_auto": k3c, "vp_lookahead": vp(0), "vp_delay1": vp(2)}
times = {k: [] for k in cases}
for r in range(4):
    for k, f in cases.items():
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        if r:
            times[k].append(e0.elapsed_time(e1))
for k in cases:
    cases[k]()
    plan = G.grpo_async_last_plan()
    ms = float(np.median(times[k]))
    print(json.dumps({"case": k, "V": V, "rows": R, "ms": round(ms, 3),
                      "frac": round((4 * V + 29) * R / ms / 1e6 / PEAK, 3), "plan": plan}), flush=True)
