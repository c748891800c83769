"""Advantages from sharded rewards over NCCL (GrpoAsyncLoss.advantage_sharded): every rank
keeps only its LPT share of the trajectories; the group statistics go through two rounds
of all-reduce.  Checks, on every rank, that the result equals the replicated computation
(grpo_async_advantage on the whole batch) bit for bit (0/1 rewards: exact partial sums).

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/sharded_rewards_nccl.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_26256_b200 as G  # noqa: E402
from synth.gen import make_batch  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    out = {"world": world}
    for name in ("dapo", "prod", "large"):
        b = make_batch(name, 0)
        ids = G.lpt_partition(b.lengths, world)[rank]
        cu = np.zeros(len(ids) + 1, np.int64)
        cu[1:] = np.cumsum(b.lengths[ids])
        t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to(dt).to(dev)
        loss = G.GrpoAsyncLoss()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        adv, inv = loss.advantage_sharded(t(b.rewards[ids], torch.float32), t(b.group_ids[ids], torch.int32),
                                          t(cu, torch.int64), b.P)
        e1.record()
        torch.cuda.synchronize(dev)
        db = G.DeviceBatch.from_host(b, dev)
        adv_full, inv_full = G.GrpoAsyncLoss().advantage(db)
        same = bool(torch.equal(adv, adv_full[t(ids, torch.int64)]) and
                    torch.equal(inv, inv_full[t(ids, torch.int64)]))
        ok = torch.tensor([1 if same else 0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        out[name] = {"bitwise_equal_to_replicated": bool(ok.item()), "ms": e0.elapsed_time(e1)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
