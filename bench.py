#!/usr/bin/env python
"""bench.py -- tokens/s of the fused async-GRPO loss fwd+bwd (arxiv 2604.26256,
PAPER.md eq:grpo_async P:9-26) on B200, as a fraction of the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config prod] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   (N > 1)

One step = the whole hot path over one synthetic batch of BASELINE.json's
workload: validate (C1/C2/C3) -> group advantages -> fused log-softmax +
ratio/clip/min + segmented mean + dlogits over every response row (chunked
through a resident logits buffer) -> (N > 1) one NCCL all-reduce of the
packed fp64 partials.  Inputs are resident in HBM when the timed region
starts; the logits working set (2 x chunk_rows x V x 2 B) is far larger than
L2, so no flush is needed between steps.  Rank 0 prints one JSON line.
See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trained tokens/s of fused async-GRPO loss fwd+bwd (152k vocab), % HBM peak"
UNIT = "tokens/s"
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="prod")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--chunk-rows", type=int, default=131072)
    ap.add_argument("--kernel", type=int, default=0, help="grpo_tune_t.kernel (0 auto)")
    ap.add_argument("--cluster", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--lag", type=int, default=0, help="grpo_tune_t.lag (kernel 3: free ring slots)")
    ap.add_argument("--chunk-kb", type=int, default=0, help="grpo_tune_t.chunk_kb (kernel 3)")
    ap.add_argument("--prefetch", type=int, default=0,
                    help="grpo_tune_t.prefetch (kernel 3: look-ahead chunks, -1 none, 0 default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target duration of the cpu_baseline oracle sample")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy_ read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        self.gpus = ",".join(str(g) for g in gpus)

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", self.gpus, f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# ------------------------------------------------------------------ reference arm (the oracle)
def oracle_sample(batch, target_rows):
    """Whole trajectories covering the first >= target_rows rows of the batch."""
    cu = batch.cu_seqlens
    n_traj = int(np.searchsorted(cu, target_rows, side="left"))
    n_traj = max(1, min(n_traj, batch.N))
    return np.arange(int(cu[n_traj]), dtype=np.int64), n_traj


def oracle_step(O, batch, rows, bits, eps):
    """The oracle's whole path on the sample: validate + advantage over the batch, rows fwd+bwd, J."""
    O.validate(batch.version_ids, batch.cu_seqlens, batch.group_ids, batch.target_ids,
               P=batch.P, V=batch.V, G=batch.G, tbs=batch.tbs, v_theta=batch.v_theta, K=batch.K,
               token_version=batch.token_version, logp_behav=batch.logp_behav)
    adv, inv, _ = O.advantage(batch.rewards, batch.group_ids, batch.cu_seqlens, batch.P)
    rr = O.rows(rows, bits, batch.V, batch.target_ids[rows], batch.logp_behav[rows],
                batch.cu_seqlens, adv, inv, eps, 1.0, want_dlogits=True)
    return rr


def load_oracle():
    # all host cores (torchrun exports OMP_NUM_THREADS=1 to its workers)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    os.environ["OMP_NUM_THREADS"] = str(cores or 1)
    import oracle.oracle as O
    return O, int(os.environ["OMP_NUM_THREADS"])


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(batch, seconds, block=512):
    """The oracle (fp64, all host cores) timed on whole trajectories covering the first
    >= 8192 rows of the batch, in blocks of `block` rows, repeated for
    ~`seconds`; plus a single-core figure on the first 1024 rows.  Input generation (the
    logits' bf16 bits) happens before the timer."""
    O, cores = load_oracle()
    rows, n_traj = oracle_sample(batch, 8192)
    blocks = [rows[i:i + block] for i in range(0, len(rows), block)]
    bits = [batch.logits_bits(b) for b in blocks]

    def one_pass(n_blocks):
        O.validate(batch.version_ids, batch.cu_seqlens, batch.group_ids, batch.target_ids,
                   P=batch.P, V=batch.V, G=batch.G, tbs=batch.tbs, v_theta=batch.v_theta, K=batch.K,
                   token_version=batch.token_version, logp_behav=batch.logp_behav)
        adv, inv, _ = O.advantage(batch.rewards, batch.group_ids, batch.cu_seqlens, batch.P)
        for b, bb in zip(blocks[:n_blocks], bits[:n_blocks]):
            O.rows(b, bb, batch.V, batch.target_ids[b], batch.logp_behav[b], batch.cu_seqlens,
                   adv, inv, 0.2, 1.0, want_dlogits=True)
        return sum(len(b) for b in blocks[:n_blocks])

    O.rows(blocks[0][:4], bits[0][:4], batch.V, batch.target_ids[blocks[0][:4]],
           batch.logp_behav[blocks[0][:4]], batch.cu_seqlens,
           np.zeros(batch.N), np.zeros(batch.N), 0.2, 1.0)   # load / warm
    t0 = time.perf_counter()
    n = reps = 0
    while True:
        n += one_pass(len(blocks))
        reps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    single = None
    try:  # the same OpenMP runtime the oracle library uses, limited to one thread
        import ctypes
        gomp = ctypes.CDLL("libgomp.so.1")
        gomp.omp_set_num_threads(1)
        t1 = time.perf_counter()
        n1 = one_pass(2)
        single = n1 / (time.perf_counter() - t1)
        gomp.omp_set_num_threads(cores)
    except OSError:
        pass
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "single_core_value": single,
            "sample": f"{len(rows)} rows (whole trajectories covering the first 8192 rows of "
                      f"'{batch.cfg.name}', V={batch.V}, {n_traj} trajectories) x {reps} "
                      f"repetitions, fwd+bwd fp64 incl. validate+advantage over the full batch; "
                      f"{dt:.1f} s; single core: the first {sum(len(b) for b in blocks[:2])} rows"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth.gen import CONFIGS, make_batch
    cfg = CONFIGS[args.config]
    batch = make_batch(cfg, args.seed, period=args.chunk_rows)
    O, cores = load_oracle()
    rows, _ = oracle_sample(batch, 256)
    bits = batch.logits_bits(rows)
    for _ in range(args.warmup):
        oracle_step(O, batch, rows, bits, cfg.eps)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(O, batch, rows, bits, cfg.eps)
    dt = time.perf_counter() - t0
    value = len(rows) * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "vocab": batch.V,
                       "sample_rows_per_step": len(rows), "tokens_per_batch": batch.T},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{len(rows)} rows per step (whole trajectories covering "
                                       f"the first 256 rows of '{args.config}'), fwd+bwd fp64 "
                                       "incl. validate+advantage over the full batch"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2604_26256_b200 as G
    import synth.gpu as SG
    from synth.gen import CONFIGS, make_batch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = CONFIGS[args.config]
    R_cfg = args.chunk_rows
    batch = make_batch(cfg, args.seed, period=R_cfg)
    V, ld = batch.V, batch.ld

    # ---- shard: token-balanced, trajectory-atomic LPT (trajectory metadata replicated)
    if world > 1:
        parts = G.lpt_partition(batch.lengths, world)
        mine = parts[rank]
    else:
        mine = np.arange(batch.N)
    rows_g, local_cu = G.shard_rows(batch.cu_seqlens, mine)
    T_local = len(rows_g)
    R = min(R_cfg, T_local)
    n_chunks = (T_local + R - 1) // R

    # ---- host inputs (pinned) and their device copies
    def pinned(x, dt):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dt).pin_memory()

    # replicated O(N) trajectory metadata + this rank's token arrays only
    host = {
        "cu": pinned(batch.cu_seqlens, torch.int64), "gid": pinned(batch.group_ids, torch.int32),
        "ver": pinned(batch.version_ids, torch.int64), "rew": pinned(batch.rewards, torch.float32),
        "tgt_l": pinned(batch.target_ids[rows_g], torch.int64),
        "lw_l": pinned(batch.logp_behav[rows_g], torch.float32),
        "cu_l": pinned(local_cu, torch.int64), "tix": pinned(mine.astype(np.int32), torch.int32),
    }
    if batch.token_version is not None:
        host["tv_l"] = pinned(batch.token_version[rows_g], torch.int64)
    d = {k: v.to(dev) for k, v in host.items()}

    def sharded(dd):
        return G.ShardedBatch(batch.P, batch.G, batch.K, V, ld, batch.tbs, batch.v_theta, batch.T,
                              dd["cu"], dd["gid"], dd["ver"], dd["rew"], dd["cu_l"], dd["tix"],
                              dd["tgt_l"], dd["lw_l"], dd.get("tv_l"))
    sb = sharded(d)

    # ---- logits (device-generated, bit-identical to synth/gen.py) and the dlogits buffer.
    # The recipe: logical row t reads physical row t % chunk_rows.  One rank holds one resident
    # chunk buffer, which is exactly every chunk's logits.  With N > 1 ranks a rank's rows are
    # a scattered set of trajectories, so each rank holds all of ITS rows' logits resident
    # (filled once, trajectory by trajectory, with the same recipe) and writes dlogits through
    # a chunk buffer sized to the memory left: every rank computes on the batch's own logits
    # and J is the unsharded batch's at every N.
    spec = batch.logits
    resident_ok = world > 1 and T_local * ld * 2 <= torch.cuda.mem_get_info(dev)[0] - (24 << 30)
    if not resident_ok:   # one rank, or a shard too large to hold (e.g. `large` at N = 2)
        spec.period = R
        logits = torch.empty((R, ld), dtype=torch.int16, device=dev)
        SG.fill_logits(logits, spec, 0, R, V)
        logits_desc = ("device-generated counter-hash bf16, rows periodic in the chunk buffer "
                       "(DESIGN.md input recipe)" + ("" if world == 1 else
                       "; rank-local rows read the chunk buffer periodically, so J is not the "
                       "batch's at this N"))
    else:
        logits = torch.empty((max(T_local, 1), ld), dtype=torch.int16, device=dev)
        base_dev = None
        for j, i in enumerate(mine):
            base_dev = SG.fill_logits(logits[int(local_cu[j]):int(local_cu[j + 1])], spec,
                                      int(batch.cu_seqlens[i]), int(batch.lengths[i]), V,
                                      base_dev=base_dev)
        torch.cuda.synchronize()
        free = torch.cuda.mem_get_info(dev)[0]
        R = int(max(1024, min(R, (free - (6 << 30)) // (ld * 2))))
        n_chunks = (T_local + R - 1) // R
        logits_desc = ("device-generated counter-hash bf16 (the N=1 recipe); each rank holds its "
                       "own rows' logits resident, dlogits through a chunk buffer")
    dlogits = torch.empty((R, ld), dtype=torch.int16, device=dev)

    def logits_of(b, n):
        return logits[b:b + n] if resident_ok else logits[:n]

    tune = None
    if (args.kernel or args.cluster or args.ctas_per_sm or args.stages or args.lag or args.chunk_kb
            or args.prefetch):
        tune = {"kernel": args.kernel, "cluster_size": args.cluster,
                "ctas_per_sm": args.ctas_per_sm, "stages": args.stages, "lag": args.lag,
                "chunk_kb": args.chunk_kb, "prefetch": args.prefetch}
    loss = G.GrpoAsyncLoss(eps=cfg.eps, std_floor=cfg.std_floor, tune=tune)
    vo = G.ValidateOut(batch.N, batch.P, batch.K, dev)
    adv = torch.empty(batch.N, dtype=torch.float32, device=dev)
    inv = torch.empty(batch.N, dtype=torch.float32, device=dev)
    traj_sum = torch.zeros(len(mine), dtype=torch.float64, device=dev)
    # this rank's packed fp64 partials: the loss stats, then the token-level validation counts
    NP = G.NUM_STATS + 3
    packed = torch.zeros(NP, dtype=torch.float64, device=dev)
    stats, tok_counts = packed[:G.NUM_STATS], packed[G.NUM_STATS:]
    glob = torch.zeros(NP, dtype=torch.float64, device=dev)   # the batch's, on every rank
    gathered = torch.zeros((world, NP), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def allgather(t):
        if world > 1:
            dist.all_gather_into_tensor(gathered, t)
        else:
            gathered[0].copy_(t)
        return gathered

    def step(sbx=sb):
        loss.validate_local(sbx, vo, token_counts=tok_counts)
        loss.advantage(sbx, adv, inv)
        traj_sum.zero_()
        stats.zero_()
        for c in range(n_chunks):
            b = c * R
            n = min(R, T_local - b)
            loss.loss_chunk(logits_of(b, n), b, n, sbx.target_ids[b:b + n], sbx.logp_behav[b:b + n],
                            sbx.local_cu, adv, inv, traj_sum, stats, dlogits=dlogits[:n],
                            traj_index=sbx.traj_index, V=V)
        # the path's one exchange: every rank's packed partials all-gathered, summed in rank
        # order by grpo_async_combine_ranks (bit-identical everywhere, run to run), and the
        # summed token counts completing the validation verdict
        loss.combine_ranks(packed, world, allgather=allgather, out=glob)
        loss.validate_combine(vo, glob[G.NUM_STATS:])

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    # ---- timed region (device-resident inputs)
    # the GPUs of this node's ranks (CUDA_VISIBLE_DEVICES, if set, maps them)
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    node_gpus = list(range(int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    if vis:
        node_gpus = [vis.split(",")[g] for g in node_gpus]
    sampler = ClockSampler(node_gpus) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    G.grpo_profile_enable(True)
    G.grpo_profile_collect()
    launches0 = loss.launches
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    G.grpo_profile_enable(False)
    n_traced, kern_ms = G.grpo_profile_collect()
    plan = G.grpo_async_last_plan()
    launches = loss.launches - launches0
    clocks = sampler.stop() if sampler else None
    ms_max = max_over_ranks(ms)
    kern_ms_max = max_over_ranks(kern_ms)
    stats_h = glob.cpu().numpy()
    summ = vo.summary_dict()

    T_total = batch.T
    value = T_total * args.steps / (ms_max / 1e3)
    peak, peak_src = measured_peaks()
    # algorithmic bytes of the fused kernel per row: read the bf16 row (2V), write the bf16
    # dlogits row (2V), read 16 B row metadata, write term (fp64) / logp / flag (13 B)
    bytes_per_row = 4 * V + 29
    rows_per_launch = T_local / n_chunks
    avg_launch_ms = kern_ms / max(n_traced, 1)
    achieved = bytes_per_row * rows_per_launch / (avg_launch_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if int(tr.get("V", -1)) == V and int(tr.get("plan_kernel", -1)) == int(plan["kernel"]):
            traffic = float(tr["dram_bytes_per_row"]) * rows_per_launch
    except Exception:
        pass

    # ---- end to end through the public API with host buffers (pinned H2D, D2H of the result)
    e2e = None
    if not args.no_e2e:
        keys_h2d = list(host.keys())
        dd = {k: torch.empty_like(d[k]) for k in keys_h2d}
        h2d = sum(host[k].numel() * host[k].element_size() for k in keys_h2d)
        sbx = sharded(dd)
        out_host = torch.empty(NP + len(G.SUMMARY_FIELDS), dtype=torch.float64).pin_memory()
        d2h = out_host.numel() * 8
        res_dev = torch.empty(NP + len(G.SUMMARY_FIELDS), dtype=torch.float64, device=dev)

        def e2e_step():
            for k in keys_h2d:
                dd[k].copy_(host[k], non_blocking=True)
            step(sbx)
            res_dev[:NP].copy_(glob)
            res_dev[NP:].copy_(vo.summary)
            out_host.copy_(res_dev, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        # the end-to-end result must be the device-timed run's, bit for bit
        e2e_same = bool(out_host[G.STAT_J].item() == float(stats_h[G.STAT_J]))
        e2e = {"value": T_total * args.steps / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms / args.steps, "result_matches_device_run": e2e_same,
               "note": "per step and rank: pinned H2D of the replicated trajectory metadata "
                       "(cu_seqlens, group ids, versions, rewards) and of this rank's token "
                       "arrays (targets, behaviour log-probs, token versions, local packing), "
                       "the whole path, D2H of the combined partials + validation summary; "
                       "logits are device-resident activations of the LM forward and are not "
                       "copied"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(batch, args.cpu_seconds)

    if rank == 0:
        J = float(stats_h[G.STAT_J])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": args.config, "tokens_per_step": T_total, "vocab": V,
                       "prompts": batch.P, "group_size": batch.G, "K": batch.K,
                       "chunk_rows": R, "n_chunks_per_rank": n_chunks,
                       "l2": "inputs larger than L2 (logits %.1f GB + dlogits chunk buffer %.1f GB)"
                             % (logits.numel() * 2 / 1e9, R * ld * 2 / 1e9),
                       "parallelism": f"dp{world} token-balanced LPT over trajectories",
                       "logits": logits_desc},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "frac_of_spec_8000_gbs": achieved / 8000.0,
                         "kernel": {2: "rowwise_kernel", 3: "stream_kernel"}.get(
                             plan["kernel"], str(plan["kernel"])),
                         "plan": plan,
                         "bytes_per_row": bytes_per_row, "launches": n_traced,
                         "avg_launch_ms": avg_launch_ms,
                         "kernel_share_of_step": kern_ms_max / ms_max},
            "path_hbm_frac": T_total * args.steps * (4 * V + 20) / (ms_max / 1e3) / 1e9 / peak,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
            "result": {"J": J, "loss": -J, "clip_frac": float(stats_h[G.STAT_CLIPPED] / T_total),
                       "active_frac": float(stats_h[G.STAT_ACTIVE] / T_total),
                       "rows": float(stats_h[G.STAT_ROWS]), "valid": summ["valid"],
                       "max_staleness": summ["max_staleness"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
