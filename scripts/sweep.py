"""Time the fused loss kernel over one resident chunk for several launch plans."""
import argparse, json, sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26256_b200 as G
import synth.gpu as SG
from synth.gen import make_batch, CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="prod")
ap.add_argument("--rows", type=int, default=65536)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--plans", default="")
ap.add_argument("--fwd-only", action="store_true")
ap.add_argument("--vocab", type=int, default=0, help="override the config's V (e.g. a vocab shard)")
args = ap.parse_args()
dev = torch.device("cuda:0")
try:  # the measured copy bandwidth (MEASURED_PEAKS.json), else the profiling guide's fallback
    PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    PEAK = 6650.0
import dataclasses
cfg = CONFIGS[args.config]
if args.vocab:
    cfg = dataclasses.replace(cfg, V=args.vocab)
b = make_batch(cfg, 0, period=args.rows)
R = args.rows
V, ld = b.V, b.ld
lg = torch.empty((R, ld), dtype=torch.int16, device=dev)
dl = torch.empty_like(lg)
SG.fill_logits(lg, b.logits, 0, R, V)
db = G.DeviceBatch.from_host(b, dev)
loss = G.GrpoAsyncLoss()
adv, inv = loss.advantage(db)
ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
plans = [json.loads(p) for p in args.plans.split(";")] if args.plans else [
    {}, {"kernel": 2}, {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3},
]
bytes_row = 4 * V + 29 if not args.fwd_only else 2 * V + 29
def run_once(plan):
    plan = dict(plan)
    for k, v in plan.pop("env", {}).items():  # launch-time environment knobs (experiments)
        os.environ[k] = str(v)
    loss.tune = plan
    G.grpo_profile_enable(True); G.grpo_profile_collect()
    loss.loss_chunk(lg, 0, R, db.target_ids[:R], db.logp_behav[:R], db.cu_seqlens, adv, inv, ts, st,
                    dlogits=None if args.fwd_only else dl, V=V)
    torch.cuda.synchronize()
    n, ms = G.grpo_profile_collect()
    return ms, G.grpo_async_last_plan()


times = {i: [] for i in range(len(plans))}
plans_used, errors = {}, {}
n_rounds = args.reps + 1 if args.reps > 0 else 1
# plans interleaved round by round, so slow drifts (power cap, clocks) hit every plan alike
for r in range(n_rounds):
    for i, plan in enumerate(plans):
        if i in errors:
            continue
        try:
            ms, pl = run_once(plan)
            for k in plan.get("env", {}):
                os.environ.pop(k, None)
            plans_used[i] = pl
            if r > 0 or args.reps == 0:
                times[i].append(ms)
        except Exception as e:
            errors[i] = str(e)
for i, plan in enumerate(plans):
    if i in errors:
        print(json.dumps({"tune": plan, "error": errors[i]}), flush=True)
        continue
    ms = float(np.median(times[i]))
    print(json.dumps({"tune": plan, "plan": plans_used[i], "ms": round(ms, 3),
                      "GBps": round(bytes_row * R / ms / 1e6, 1),
                      "frac": round(bytes_row * R / ms / 1e6 / PEAK, 3)}), flush=True)
G.grpo_profile_enable(False)
