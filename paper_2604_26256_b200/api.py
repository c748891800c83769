"""Python plumbing above the C ABI: device buffers for one training batch and
the order of calls of one step of the hot path (validate -> advantage ->
fused loss over row chunks).  Every numeric step runs in the CUDA kernels of
libgrpo_async.so; this module only allocates torch tensors and calls the
binding (paper_2604_26256_b200._lib).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


@dataclass
class DeviceBatch:
    """Packed batch metadata on the device (trajectories of
    up to K versions, G responses per prompt; response rows only)."""
    P: int
    G: int
    K: int
    V: int
    ld: int
    tbs: int
    v_theta: int
    cu_seqlens: torch.Tensor       # int64 [N+1]
    group_ids: torch.Tensor        # int32 [N]
    version_ids: torch.Tensor      # int64 [N]
    rewards: torch.Tensor          # float32 [N]
    target_ids: torch.Tensor       # int64 [T]
    logp_behav: torch.Tensor       # float32 [T]
    token_version: torch.Tensor | None = None  # int64 [T]

    @property
    def N(self):
        return self.group_ids.numel()

    @property
    def T(self):
        return self.target_ids.numel()

    @staticmethod
    def from_host(b, device, pin=False):
        """b: any object with the synth.gen.Batch fields (numpy arrays)."""
        def t(x, dt):
            if x is None:
                return None
            h = torch.from_numpy(np.ascontiguousarray(x)).to(dt)
            if pin:
                h = h.pin_memory()
            return h.to(device, non_blocking=pin)
        return DeviceBatch(b.P, b.G, b.K, b.V, b.ld, b.tbs, b.v_theta,
                           t(b.cu_seqlens, torch.int64), t(b.group_ids, torch.int32),
                           t(b.version_ids, torch.int64), t(b.rewards, torch.float32),
                           t(b.target_ids, torch.int64), t(b.logp_behav, torch.float32),
                           t(b.token_version, torch.int64))


@dataclass
class ShardedBatch:
    """One rank's view of a trajectory-sharded batch: the O(N) trajectory
    metadata replicated (cu_seqlens of the global packing, group ids, versions, rewards),
    the token arrays only for this rank's trajectories traj_index, in the local packing
    local_cu (trajectory j of this rank owns local rows [local_cu[j], local_cu[j+1]))."""
    P: int
    G: int
    K: int
    V: int
    ld: int
    tbs: int
    v_theta: int
    T: int                         # global row count (cu_seqlens[N])
    cu_seqlens: torch.Tensor       # int64 [N+1]
    group_ids: torch.Tensor        # int32 [N]
    version_ids: torch.Tensor      # int64 [N]
    rewards: torch.Tensor          # float32 [N]
    local_cu: torch.Tensor         # int64 [n_local+1]
    traj_index: torch.Tensor       # int32 [n_local]
    target_ids: torch.Tensor       # int64 [T_local]
    logp_behav: torch.Tensor       # float32 [T_local]
    token_version: torch.Tensor | None = None  # int64 [T_local]

    @property
    def N(self):
        return self.group_ids.numel()

    @property
    def n_local(self):
        return self.traj_index.numel()

    @property
    def T_local(self):
        return self.target_ids.numel()


class ValidateOut:
    def __init__(self, N, P, K, device):
        self.traj_flags = torch.zeros(max(N, 1), dtype=torch.int32, device=device)
        self.group_count = torch.zeros(P, dtype=torch.int32, device=device)
        self.stale_hist = torch.zeros(P * (K + 1), dtype=torch.int32, device=device)
        self.summary = torch.zeros(len(L.SUMMARY_FIELDS), dtype=torch.int64, device=device)

    def summary_dict(self):
        return dict(zip(L.SUMMARY_FIELDS, self.summary.cpu().tolist()))


class GrpoAsyncLoss:
    """One step of the hot path over a DeviceBatch.

    eps: clip range; grad_scale multiplies dlogits; std_floor: Z2.
    DAPO options: eps_hi (clip-higher upper range, default eps),
    norm ("seq" = eq:grpo_async as written, "token" = DAPO token mean), traj_mask
    (uint8 device tensor [N], 0 drops a trajectory from the loss) and std_unbiased
    (sample std, n - 1, in the group advantage).
    tune: optional dict for grpo_tune_t (kernel / cluster_size / ctas_per_sm / stages / ...).
    """

    def __init__(self, eps=0.2, std_floor=1e-8, grad_scale=1.0, tune=None, eps_hi=None,
                 norm="seq", traj_mask=None, std_unbiased=False):
        self.eps = float(eps)
        self.std_unbiased = bool(std_unbiased)
        self.eps_hi = float(eps if eps_hi is None else eps_hi)
        self.norm = {"seq": L.NORM_SEQ, "token": L.NORM_TOKEN}[norm]
        self.traj_mask = traj_mask
        self.std_floor = float(std_floor)
        self.grad_scale = float(grad_scale)
        self.tune = tune
        self._ws = None
        self.launches = 0

    # ---- validate (C1/C2/C3)
    def validate(self, db: DeviceBatch, out: ValidateOut | None = None, stream=None):
        out = out or ValidateOut(db.N, db.P, db.K, db.target_ids.device)
        L.grpo_async_validate(db.version_ids, db.token_version, db.cu_seqlens, db.group_ids,
                              db.target_ids, db.logp_behav, db.N, db.T, db.P, db.V, db.G, db.tbs,
                              db.v_theta, db.K, out.traj_flags, out.group_count, out.stale_hist,
                              out.summary, stream)
        self.launches += L.grpo_last_launch_count()
        return out

    def validate_local(self, sb: ShardedBatch, out: ValidateOut | None = None, token_counts=None,
                       stream=None):
        """One rank of a sharded batch: trajectory checks over all N, token checks over this
        rank's trajectories; token_counts (float64[3] device tensor, e.g. a slice of the packed
        partials) receives the local token-level counts."""
        out = out or ValidateOut(sb.N, sb.P, sb.K, sb.cu_seqlens.device)
        L.grpo_async_validate_local(sb.version_ids, sb.cu_seqlens, sb.group_ids, sb.N, sb.T, sb.P,
                                    sb.V, sb.G, sb.tbs, sb.v_theta, sb.K, sb.local_cu,
                                    sb.traj_index, sb.n_local, sb.token_version, sb.target_ids,
                                    sb.logp_behav, out.traj_flags, out.group_count,
                                    out.stale_hist, out.summary, token_counts, stream)
        self.launches += L.grpo_last_launch_count()
        return out

    def combine_ranks(self, packed, world, allgather=None, out=None, stream=None):
        """The data-parallel step's one exchange: all-gather every rank's packed float64
        partials and sum them in rank order on the device (deterministic, identical on every
        rank).  allgather(t) -> [world, n] (default: torch.distributed.all_gather_into_tensor)."""
        if allgather is None:
            import torch.distributed as dist

            def allgather(t):
                g = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
                dist.all_gather_into_tensor(g, t)
                return g
        gathered = allgather(packed)
        out = out if out is not None else torch.empty_like(packed)
        L.grpo_async_combine_ranks(gathered, world, packed.numel(), out, stream)
        self.launches += L.grpo_last_launch_count()
        return out

    def validate_combine(self, out: ValidateOut, token_counts, stream=None):
        L.grpo_async_validate_combine(out.summary, token_counts, stream)
        self.launches += L.grpo_last_launch_count()

    # ---- advantages, eq:group_advantage P:153-156
    def advantage(self, db: DeviceBatch, adv=None, inv_norm=None, stream=None):
        dev = db.rewards.device
        adv = adv if adv is not None else torch.empty(db.N, dtype=torch.float32, device=dev)
        inv = inv_norm if inv_norm is not None else torch.empty(db.N, dtype=torch.float32, device=dev)
        if self._default_opts():
            L.grpo_async_advantage(db.rewards, db.group_ids, db.cu_seqlens, db.N, db.P,
                                   self.std_floor, adv, inv, None, stream)
        else:
            L.grpo_async_advantage_ex(db.rewards, db.group_ids, db.cu_seqlens, db.N, db.P,
                                      self.std_floor, self.eps, self.eps_hi, self.norm,
                                      self.traj_mask, adv, inv, None, stream,
                                      std_unbiased=self.std_unbiased)
        self.launches += L.grpo_last_launch_count()
        return adv, inv

    # ---- advantages from sharded rewards (SURVEY §8e "group reward statistics" variant)
    def advantage_sharded(self, rewards, group_ids, cu_seqlens, P, allreduce=None, stream=None):
        """This rank's trajectories only (rewards, group_ids, local cu_seqlens); the group
        statistics of all ranks are combined with two rounds of all-reduce.  `allreduce(t, op)`
        reduces a float64 device tensor in place over the ranks ("sum" or "max"); the default
        uses torch.distributed (NCCL).  Returns (adv, inv_norm) of the local trajectories."""
        if allreduce is None:
            import torch.distributed as dist

            def allreduce(t, op):
                dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)
        dev = rewards.device
        N = int(rewards.numel())
        part = torch.empty(4 * P + 1, dtype=torch.float64, device=dev)
        L.grpo_async_group_partials(rewards, group_ids, cu_seqlens, N, P, part, self.traj_mask,
                                    stream)
        self.launches += L.grpo_last_launch_count()
        p4 = part[:4 * P].view(P, 4)
        summed = torch.cat([p4[:, :2].reshape(-1), part[4 * P:]])
        maxed = p4[:, 2:].reshape(-1).contiguous()
        allreduce(summed, "sum")
        allreduce(maxed, "max")
        glob = torch.empty_like(part)
        g4 = glob[:4 * P].view(P, 4)
        g4[:, :2] = summed[:2 * P].view(P, 2)
        g4[:, 2:] = maxed.view(P, 2)
        glob[4 * P] = summed[2 * P]
        ss = torch.empty(P, dtype=torch.float64, device=dev)
        L.grpo_async_group_sq_partials(rewards, group_ids, N, P, glob, ss, stream)
        self.launches += L.grpo_last_launch_count()
        allreduce(ss, "sum")
        adv = torch.empty(max(N, 1), dtype=torch.float32, device=dev)
        inv = torch.empty(max(N, 1), dtype=torch.float32, device=dev)
        L.grpo_async_advantage_from_stats(rewards, group_ids, cu_seqlens, N, P, self.std_floor,
                                          self.norm, self.traj_mask, self.std_unbiased, glob, ss,
                                          adv, inv, stream)
        self.launches += L.grpo_last_launch_count()
        return adv[:N], inv[:N]

    def _default_opts(self):
        return (self.eps_hi == self.eps and self.norm == L.NORM_SEQ and self.traj_mask is None
                and not self.std_unbiased)

    def workspace(self, n_rows, V, N, device):
        need = L.grpo_async_workspace_size(n_rows, V, N)
        if self._ws is None or self._ws.numel() < need or self._ws.device != device:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    # ---- fused loss fwd (+ bwd when dlogits is given), eq:grpo_async P:9-26
    def loss_chunk(self, logits, row_begin, n_rows, target_ids, logp_behav, cu_seqlens, adv,
                   inv_norm, traj_sum, stats, dlogits=None, traj_index=None, logp_out=None,
                   lse_out=None, scale_out=None, V=None, stream=None):
        V = V if V is not None else logits.shape[1]
        ld = logits.shape[1]
        N = cu_seqlens.numel() - 1
        ws = self.workspace(n_rows, V, N, logits.device)
        if self._default_opts():
            L.grpo_async_loss_fwd(logits, row_begin, n_rows, V, ld, target_ids, logp_behav,
                                  cu_seqlens, N, traj_index, adv, inv_norm, self.eps,
                                  self.grad_scale, logp_out, lse_out, scale_out, traj_sum, stats,
                                  dlogits, ws, self.tune, stream)
        else:
            L.grpo_async_loss_fwd_ex(logits, row_begin, n_rows, V, ld, target_ids, logp_behav,
                                     cu_seqlens, N, traj_index, adv, inv_norm, self.eps,
                                     self.eps_hi, self.norm, self.traj_mask, self.grad_scale,
                                     logp_out, lse_out, scale_out, traj_sum, stats, dlogits, ws,
                                     self.tune, stream)
        self.launches += L.grpo_last_launch_count()

    # ---- LM-head-fused loss: logits = hidden W^T on the tensor cores
    def lmhead_workspace(self, n_rows, V, N, device):
        need = L.grpo_async_lmhead_workspace_size(n_rows, V, N)
        if self._ws is None or self._ws.numel() < need or self._ws.device != device:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    def lmhead_fwd(self, hidden, W, row_begin, n_rows, target_ids, logp_behav, cu_seqlens, adv,
                   inv_norm, traj_sum, stats, traj_index=None, logp_out=None, lse_out=None,
                   scale_out=None, stream=None):
        """hidden bf16 [n_rows, d], W bf16 [V, d]; outputs as loss_chunk (no logits in HBM)."""
        V, d = W.shape
        N = cu_seqlens.numel() - 1
        ws = self.lmhead_workspace(n_rows, V, N, W.device)
        L.grpo_async_lmhead_fwd(hidden, W, row_begin, n_rows, d, V, target_ids, logp_behav,
                                cu_seqlens, N, traj_index, adv, inv_norm, self.eps, self.eps_hi,
                                self.norm, self.traj_mask, self.grad_scale, logp_out, lse_out,
                                scale_out, traj_sum, stats, ws, stream)
        self.launches += L.grpo_last_launch_count()

    def lmhead_bwd(self, hidden, W, n_rows, target_ids, lse, token_scale, dz, dhidden=None,
                   dW=None, mult=1.0, stream=None):
        """dz bf16 [n_rows, ld_dz] (written), dhidden bf16 [n_rows, d] (written), dW f32 [V, d]
        (accumulated)."""
        V, d = W.shape
        L.grpo_async_lmhead_bwd(hidden, W, n_rows, d, V, target_ids, lse, token_scale, mult, dz,
                                dz.shape[1], dhidden, dW, stream)
        self.launches += L.grpo_last_launch_count()

    # ---- tensor-parallel LM head: W split by vocabulary rows over the ranks of a group
    def lmhead_tp_fwd(self, hidden, W_shard, col_offset, V, row_begin, n_rows, target_ids,
                      logp_behav, cu_seqlens, adv, inv_norm, traj_sum, stats, allgather=None,
                      R=None, logp_out=None, lse_out=None, scale_out=None, traj_index=None,
                      stream=None):
        """allgather(t) returns the ranks' copies of the float32 device tensor t stacked in
        rank order (default: torch.distributed.all_gather_into_tensor over NCCL)."""
        Vs, d = W_shard.shape
        dev = W_shard.device
        ws = torch.empty(L.grpo_async_lmhead_workspace_size(n_rows, Vs, 1), dtype=torch.uint8,
                         device=dev)
        part = torch.empty((max(n_rows, 1), 4), dtype=torch.float32, device=dev)
        L.grpo_async_lmhead_tp_partials(hidden, W_shard, n_rows, d, Vs, col_offset, target_ids,
                                        part, ws, stream)
        self.launches += L.grpo_last_launch_count()
        if allgather is None:
            import torch.distributed as dist

            def allgather(t):
                out = torch.empty((dist.get_world_size(),) + tuple(t.shape), dtype=t.dtype,
                                  device=t.device)
                dist.all_gather_into_tensor(out, t.contiguous())
                return out
        parts = allgather(part).contiguous()
        R = parts.shape[0]
        N = cu_seqlens.numel() - 1
        ws2 = self.workspace(n_rows, V, N, dev)
        L.grpo_async_lmhead_tp_fwd(parts, R, row_begin, n_rows, V, target_ids, logp_behav,
                                   cu_seqlens, N, traj_index, adv, inv_norm, self.eps, self.eps_hi,
                                   self.norm, self.traj_mask, self.grad_scale, logp_out, lse_out,
                                   scale_out, traj_sum, stats, ws2, stream)
        self.launches += L.grpo_last_launch_count()

    def lmhead_tp_bwd(self, hidden, W_shard, col_offset, n_rows, target_ids, lse, token_scale, dz,
                      dhidden_partial=None, dW_shard=None, mult=1.0, stream=None,
                      allreduce_async=None):
        """dhidden_partial (float32) is this shard's dz W_shard: sum it over the ranks.  With
        allreduce_async(t) -> handle (e.g. torch.distributed.all_reduce(t, async_op=True)) the
        all-reduce of dhidden_partial is started right after its GEMM and overlaps the dW GEMM;
        the handle is returned (wait() before using dhidden_partial)."""
        Vs, d = W_shard.shape
        if allreduce_async is None:
            L.grpo_async_lmhead_tp_bwd(hidden, W_shard, n_rows, d, Vs, col_offset, target_ids, lse,
                                       token_scale, mult, dz, dz.shape[1], dhidden_partial,
                                       dW_shard, stream)
            self.launches += L.grpo_last_launch_count()
            return None
        L.grpo_async_lmhead_tp_bwd(hidden, W_shard, n_rows, d, Vs, col_offset, target_ids, lse,
                                   token_scale, mult, dz, dz.shape[1], dhidden_partial, None, stream)
        self.launches += L.grpo_last_launch_count()
        handle = allreduce_async(dhidden_partial)
        if dW_shard is not None:
            L.grpo_async_lmhead_dw(hidden, n_rows, d, Vs, dz, dz.shape[1], dW_shard, stream)
        return handle

    # ---- fused loss over vocabulary-parallel logits
    def loss_chunk_vp(self, comm, shards, row_begin, n_rows, target_ids, logp_behav, cu_seqlens,
                      adv, inv_norm, traj_sum, stats, dshards=None, traj_index=None,
                      logp_out=None, lse_out=None, scale_out=None, V=None, stream=None):
        """comm: VpGroup; shards / dshards: this process's local shard tensors [n_rows, ld]."""
        ld = shards[0].shape[1]
        N = cu_seqlens.numel() - 1
        V = V if V is not None else comm.world * comm.shard_cols
        ws = self.workspace(n_rows, V, N, shards[0].device)
        try:
            L.grpo_async_loss_fwd_vp(comm.world, comm.rank_begin, comm.shard_cols, comm.slots,
                                     shards, dshards,
                                     comm.xbuf, comm.epoch, row_begin, n_rows, V, ld,
                                     target_ids, logp_behav, cu_seqlens, N, traj_index, adv,
                                     inv_norm, self.eps, self.eps_hi, self.norm, self.traj_mask,
                                     self.grad_scale, logp_out, lse_out, scale_out, traj_sum,
                                     stats, ws, stream, lag=comm.lag, dynamic_rows=comm.dynamic_rows)
        finally:
            # every call consumes an epoch on every rank, even one this rank refused on the
            # host: the ranks' epochs (exchange-buffer halves and tags) stay in step
            comm.epoch += 1
        self.launches += L.grpo_last_launch_count()

    def loss_bwd(self, logits, n_rows, V, target_ids, lse, token_scale, dlogits, mult=1.0,
                 stream=None):
        L.grpo_async_loss_bwd(logits, n_rows, V, logits.shape[1], target_ids, lse, token_scale,
                              mult, dlogits, stream)
        self.launches += L.grpo_last_launch_count()


class VpGroup:
    """Exchange buffers of a vocabulary-parallel group (grpo_vp_comm_t without the logits).

    xbuf[q] (2 * slots * world * 32 B, zeroed once) belongs to rank q (slots = the most
    rows one call may process; two halves so that consecutive calls never share a
    slot); every process holds all `world` addresses (its own plus peer mappings).
    `local(...)` builds the single-GPU group in which one process runs all ranks;
    `from_symmetric(...)` maps the buffers of a torch.distributed group through torch
    symmetric memory (NVLink peer pointers).  epoch counts the calls made.
    """

    def __init__(self, world, rank_begin, shard_cols, slots, xbuf, keep=()):
        self.world, self.rank_begin, self.shard_cols = world, rank_begin, shard_cols
        self.slots = slots
        self.lag = 0              # grpo_vp_comm_t.lag
        self.dynamic_rows = 0     # grpo_vp_comm_t.dynamic_rows
        self.xbuf = list(xbuf)
        self.epoch = 0
        self._keep = keep

    @staticmethod
    def shard_cols_for(V, world):
        return -(-V // (world * 8)) * 8

    @staticmethod
    def _words(slots, world):
        return 2 * slots * world * 4  # int64 words

    @staticmethod
    def local(world, V, max_rows, device, shard_cols=None):
        sc = shard_cols or VpGroup.shard_cols_for(V, world)
        slots = max(max_rows, 1)
        xb = [torch.zeros(VpGroup._words(slots, world), dtype=torch.int64, device=device)
              for _ in range(world)]
        return VpGroup(world, 0, sc, slots, [x.data_ptr() for x in xb], keep=(xb,))

    @staticmethod
    def from_symmetric(V, max_rows, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        sc = VpGroup.shard_cols_for(V, world)
        slots = max(max_rows, 1)
        n = VpGroup._words(slots, world)
        buf = symm.empty(n, dtype=torch.int64, device=device)
        buf.zero_()
        h = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
        xb = [h.get_buffer(q, (n,), torch.int64).data_ptr() for q in range(world)]
        torch.cuda.synchronize(device)
        dist.barrier(group)
        return VpGroup(world, rank, sc, slots, xb, keep=(buf, h))


def lpt_partition(lengths, world_size):
    """Token-balanced, trajectory-atomic partition (longest processing time first).

    Sort trajectories by length descending (ties: lower index first) and give
    each to the currently least-loaded rank (ties: lower rank).  Returns a list
    of ascending index arrays, one per rank.  Long-tailed lengths make a
    count-balanced split skewed.
    """
    lengths = np.asarray(lengths, np.int64)
    order = np.lexsort((np.arange(len(lengths)), -lengths))
    load = np.zeros(world_size, np.int64)
    owner = np.empty(len(lengths), np.int64)
    for i in order:
        r = int(np.argmin(load))          # argmin returns the lowest rank on ties
        owner[i] = r
        load[r] += lengths[i]
    return [np.nonzero(owner == r)[0] for r in range(world_size)]


def shard_rows(cu_seqlens, traj_ids):
    """Global row indices of the given trajectories, in order, and the local cu_seqlens."""
    cu = np.asarray(cu_seqlens, np.int64)
    L_ = cu[1:] - cu[:-1]
    Ls = L_[traj_ids]
    local_cu = np.zeros(len(traj_ids) + 1, np.int64)
    local_cu[1:] = np.cumsum(Ls)
    rows = np.concatenate([np.arange(cu[i], cu[i + 1]) for i in traj_ids]) if len(traj_ids) else \
        np.zeros(0, np.int64)
    return rows, local_cu
