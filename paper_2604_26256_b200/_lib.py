"""Thin ctypes binding of include/grpo_async.h (argument marshalling only).

Every function here has the name of the C entry point it calls and does
nothing but turn torch device tensors into pointers, pick the current CUDA
stream, and raise on a non-OK status.  All arithmetic happens in the CUDA
kernels of libgrpo_async.so.  There is no fallback: if the library is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgrpo_async.so")

GRPO_OK, GRPO_ERR_VALIDATION, GRPO_ERR_INVALID_ARG, GRPO_ERR_ALIGNMENT, GRPO_ERR_WORKSPACE, \
    GRPO_ERR_CUDA = range(6)
STATUS_NAMES = ["OK", "VALIDATION", "INVALID_ARG", "ALIGNMENT", "WORKSPACE", "CUDA"]

FLAG_NAMES = ["STALE", "FUTURE", "ZERO_LEN", "BAD_GROUP_ID", "GROUP_SIZE", "C1_MIXED",
              "BAD_TARGET", "BAD_LOGP_BEHAV"]
STAT_J, STAT_ROWS, STAT_CLIPPED, STAT_ACTIVE, STAT_ABS, STAT_LOGP = range(6)
NUM_STATS = 6

SUMMARY_FIELDS = ("n_traj", "n_tokens", "n_stale", "n_future", "n_zero_len", "n_bad_group_id",
                  "n_group_size", "n_c1_mixed", "n_bad_target", "n_bad_logp_behav",
                  "n_groups_wrong_size", "c2_dropped", "max_staleness", "min_staleness",
                  "cu_ok", "tbs_ok", "c1_ok", "c2_ok", "c3_ok", "valid")

EXPORTED = ("grpo_async_validate", "grpo_async_validate_sync", "grpo_async_validate_local",
            "grpo_async_validate_combine", "grpo_async_combine_ranks", "grpo_async_advantage",
            "grpo_async_advantage_ex", "grpo_async_loss_fwd", "grpo_async_loss_fwd_ex",
            "grpo_async_loss_fwd_vp", "grpo_async_loss_bwd", "grpo_async_workspace_size",
            "grpo_async_lmhead_workspace_size", "grpo_async_lmhead_fwd", "grpo_async_lmhead_bwd",
            "grpo_async_lmhead_logits", "grpo_async_lmhead_set_cta_group",
            "grpo_async_group_partials", "grpo_async_group_sq_partials",
            "grpo_async_advantage_from_stats", "grpo_async_lmhead_tp_partials",
            "grpo_async_lmhead_tp_fwd", "grpo_async_lmhead_tp_bwd", "grpo_async_lmhead_dw",
            "grpo_async_lmhead_tp_dx", "grpo_async_lmhead_tp_dx_reduce", "grpo_async_lmhead_dx",
            "grpo_profile_enable", "grpo_profile_collect", "grpo_async_last_plan",
            "grpo_last_launch_count",
            "grpo_last_error", "grpo_version")


class ValidateSummary(C.Structure):
    _fields_ = [(n, C.c_int64) for n in SUMMARY_FIELDS]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n in SUMMARY_FIELDS}


class Tune(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("cluster_size", C.c_int32),
                ("ctas_per_sm", C.c_int32), ("stages", C.c_int32), ("lag", C.c_int32),
                ("prefetch", C.c_int32), ("row_cache", C.c_int32), ("chunk_kb", C.c_int32)]


NORM_SEQ, NORM_TOKEN = 0, 1


class LossOpts(C.Structure):
    _fields_ = [("eps_lo", C.c_float), ("eps_hi", C.c_float), ("norm", C.c_int32),
                ("traj_mask", C.c_void_p), ("std_unbiased", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kernel", "cluster_size", "ctas_per_sm", "stages",
                                         "vec_per_thread", "grid", "max_clusters", "smem_bytes", "lag")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


VP_MAX_RANKS = 8


class VpComm(C.Structure):
    """grpo_vp_comm_t: the vocabulary-parallel group (device pointers as integers)."""
    _fields_ = [("world", C.c_int32), ("rank_begin", C.c_int32), ("n_local", C.c_int32),
                ("shard_cols", C.c_int32), ("slots", C.c_int64), ("logits", C.c_void_p * VP_MAX_RANKS),
                ("dlogits", C.c_void_p * VP_MAX_RANKS), ("xbuf", C.c_void_p * VP_MAX_RANKS),
                ("epoch", C.c_uint32), ("lag", C.c_int32), ("dynamic_rows", C.c_int32)]


class GrpoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 6 else status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python "
                          "paper_2604_26256_b200/build.py` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, i32, i64, f32, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_size_t
    st = C.c_int
    lib.grpo_async_validate.argtypes = [P, P, P, P, P, P, i32, i64, i32, i32, i32, i32, i64, i32,
                                        P, P, P, P, P]
    lib.grpo_async_validate.restype = st
    lib.grpo_async_validate_sync.argtypes = [P, P, P, P, P, P, i32, i64, i32, i32, i32, i32, i64,
                                             i32, P, P, P, P, P, P]
    lib.grpo_async_validate_sync.restype = st
    lib.grpo_async_validate_local.argtypes = [P, P, P, i32, i64, i32, i32, i32, i32, i64, i32,
                                              P, P, i32, P, P, P, P, P, P, P, P, P]
    lib.grpo_async_validate_local.restype = st
    lib.grpo_async_validate_combine.argtypes = [P, P, P]
    lib.grpo_async_validate_combine.restype = st
    lib.grpo_async_combine_ranks.argtypes = [P, i32, i32, P, P]
    lib.grpo_async_combine_ranks.restype = st
    lib.grpo_async_advantage.argtypes = [P, P, P, i32, i32, f32, P, P, P, P]
    lib.grpo_async_advantage.restype = st
    lib.grpo_async_loss_fwd.argtypes = [P, i64, i64, i32, i64, P, P, P, i32, P, P, P, f32, f32,
                                        P, P, P, P, P, P, P, sz, P, P]
    lib.grpo_async_loss_fwd.restype = st
    lib.grpo_async_advantage_ex.argtypes = [P, P, P, i32, i32, f32, P, P, P, P, P]
    lib.grpo_async_advantage_ex.restype = st
    lib.grpo_async_loss_fwd_ex.argtypes = [P, i64, i64, i32, i64, P, P, P, i32, P, P, P, P, f32,
                                           P, P, P, P, P, P, P, sz, P, P]
    lib.grpo_async_loss_fwd_ex.restype = st
    lib.grpo_async_loss_fwd_vp.argtypes = [P, i64, i64, i32, i64, P, P, P, i32, P, P, P, P, f32,
                                           P, P, P, P, P, P, sz, P]
    lib.grpo_async_loss_fwd_vp.restype = st
    lib.grpo_async_lmhead_workspace_size.argtypes = [i64, i32, i32]
    lib.grpo_async_lmhead_workspace_size.restype = sz
    lib.grpo_async_lmhead_fwd.argtypes = [P, P, i64, i64, i32, i32, P, P, P, i32, P, P, P, P, f32,
                                          P, P, P, P, P, P, sz, P]
    lib.grpo_async_lmhead_fwd.restype = st
    lib.grpo_async_lmhead_bwd.argtypes = [P, P, i64, i32, i32, P, P, P, f32, P, i64, P, P, P]
    lib.grpo_async_lmhead_bwd.restype = st
    lib.grpo_async_lmhead_logits.argtypes = [P, P, i64, i32, i32, P, i64, P]
    lib.grpo_async_lmhead_logits.restype = st
    lib.grpo_async_group_partials.argtypes = [P, P, P, i32, i32, P, P, P]
    lib.grpo_async_group_partials.restype = st
    lib.grpo_async_group_sq_partials.argtypes = [P, P, i32, i32, P, P, P]
    lib.grpo_async_group_sq_partials.restype = st
    lib.grpo_async_advantage_from_stats.argtypes = [P, P, P, i32, i32, f32, P, P, P, P, P, P]
    lib.grpo_async_advantage_from_stats.restype = st
    lib.grpo_async_lmhead_tp_partials.argtypes = [P, P, i64, i32, i32, i32, P, P, P, sz, P]
    lib.grpo_async_lmhead_tp_partials.restype = st
    lib.grpo_async_lmhead_tp_fwd.argtypes = [P, i32, i64, i64, i32, P, P, P, i32, P, P, P, P, f32,
                                             P, P, P, P, P, P, sz, P]
    lib.grpo_async_lmhead_tp_fwd.restype = st
    lib.grpo_async_lmhead_tp_bwd.argtypes = [P, P, i64, i32, i32, i32, P, P, P, f32, P, i64, P, P, P]
    lib.grpo_async_lmhead_tp_bwd.restype = st
    lib.grpo_async_lmhead_tp_dx.argtypes = [P, i64, P, i64, i32, i32, i32, i32, P, C.c_uint32, P]
    lib.grpo_async_lmhead_tp_dx.restype = st
    lib.grpo_async_lmhead_tp_dx_reduce.argtypes = [P, i32, i64, i32, i32, P, i32, C.c_uint32, P]
    lib.grpo_async_lmhead_tp_dx_reduce.restype = st
    lib.grpo_async_lmhead_dw.argtypes = [P, i64, i32, i32, P, i64, P, P]
    lib.grpo_async_lmhead_dx.argtypes = [P, i64, P, i64, i32, i32, P, i32, P]
    lib.grpo_async_lmhead_dx.restype = st
    lib.grpo_async_lmhead_dw.restype = st
    lib.grpo_async_lmhead_set_cta_group.argtypes = [i32]
    lib.grpo_async_lmhead_set_cta_group.restype = st
    lib.grpo_async_loss_bwd.argtypes = [P, i64, i32, i64, P, P, P, f32, P, P]
    lib.grpo_async_loss_bwd.restype = st
    lib.grpo_async_workspace_size.argtypes = [i64, i32, i32]
    lib.grpo_async_workspace_size.restype = sz
    lib.grpo_profile_enable.argtypes = [i32]
    lib.grpo_profile_enable.restype = st
    lib.grpo_profile_collect.argtypes = [P, P]
    lib.grpo_profile_collect.restype = st
    lib.grpo_async_last_plan.argtypes = [P]
    lib.grpo_async_last_plan.restype = st
    lib.grpo_last_launch_count.argtypes = []
    lib.grpo_last_launch_count.restype = i32
    lib.grpo_last_error.argtypes = []
    lib.grpo_last_error.restype = C.c_char_p
    lib.grpo_version.argtypes = []
    lib.grpo_version.restype = C.c_char_p
    return lib


LIB = _load()


def _ptr(t, dtype=None, name="tensor"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(status):
    if status != GRPO_OK:
        raise GrpoError(status, LIB.grpo_last_error().decode())


def grpo_profile_enable(on: bool) -> None:
    _check(LIB.grpo_profile_enable(1 if on else 0))


def grpo_profile_collect():
    """(launches traced since the last collect, their total duration in ms)."""
    n = C.c_int32()
    ms = C.c_double()
    _check(LIB.grpo_profile_collect(C.byref(n), C.byref(ms)))
    return int(n.value), float(ms.value)


def grpo_async_last_plan() -> dict:
    p = Plan()
    _check(LIB.grpo_async_last_plan(C.byref(p)))
    return p.as_dict()


def grpo_last_launch_count() -> int:
    return int(LIB.grpo_last_launch_count())


def grpo_last_error() -> str:
    return LIB.grpo_last_error().decode()


def grpo_version() -> str:
    return LIB.grpo_version().decode()


def grpo_async_workspace_size(n_rows: int, V: int, N: int) -> int:
    return int(LIB.grpo_async_workspace_size(n_rows, V, N))


def grpo_async_validate(version_ids, token_version, cu_seqlens, group_ids, target_ids, logp_behav,
                        N, T, P, V, G, tbs, v_theta, K, traj_flags, group_count, stale_hist,
                        summary, stream=None):
    """summary: int64 device tensor of len(SUMMARY_FIELDS)."""
    _check(LIB.grpo_async_validate(
        _ptr(version_ids, torch.int64, "version_ids"), _ptr(token_version, torch.int64, "token_version"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), _ptr(group_ids, torch.int32, "group_ids"),
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(logp_behav, torch.float32, "logp_behav"),
        N, T, P, V, G, tbs, v_theta, K, _ptr(traj_flags, torch.int32, "traj_flags"),
        _ptr(group_count, torch.int32, "group_count"), _ptr(stale_hist, torch.int32, "stale_hist"),
        _ptr(summary, torch.int64, "summary"), _stream(stream)))


def grpo_async_validate_local(version_ids, cu_seqlens, group_ids, N, T, P, V, G, tbs, v_theta, K,
                              local_cu, traj_index, n_local, token_version_local, target_ids_local,
                              logp_behav_local, traj_flags, group_count, stale_hist, summary,
                              token_counts=None, stream=None):
    """One rank of a trajectory-sharded batch: trajectory checks over all N, token checks over
    the n_local trajectories traj_index (local packing local_cu); token_counts: float64[3]."""
    _check(LIB.grpo_async_validate_local(
        _ptr(version_ids, torch.int64, "version_ids"), _ptr(cu_seqlens, torch.int64, "cu_seqlens"),
        _ptr(group_ids, torch.int32, "group_ids"), N, T, P, V, G, tbs, v_theta, K,
        _ptr(local_cu, torch.int64, "local_cu"), _ptr(traj_index, torch.int32, "traj_index"), n_local,
        _ptr(token_version_local, torch.int64, "token_version_local"),
        _ptr(target_ids_local, torch.int64, "target_ids_local"),
        _ptr(logp_behav_local, torch.float32, "logp_behav_local"),
        _ptr(traj_flags, torch.int32, "traj_flags"), _ptr(group_count, torch.int32, "group_count"),
        _ptr(stale_hist, torch.int32, "stale_hist"), _ptr(summary, torch.int64, "summary"),
        _ptr(token_counts, torch.float64, "token_counts"), _stream(stream)))


def grpo_async_validate_combine(summary, token_counts, stream=None):
    _check(LIB.grpo_async_validate_combine(_ptr(summary, torch.int64, "summary"),
                                           _ptr(token_counts, torch.float64, "token_counts"),
                                           _stream(stream)))


def grpo_async_combine_ranks(gathered, world, n, out, stream=None):
    """out[k] = sum over ranks in rank order of gathered[q, k] (float64 device tensors)."""
    _check(LIB.grpo_async_combine_ranks(_ptr(gathered, torch.float64, "gathered"), world, n,
                                        _ptr(out, torch.float64, "out"), _stream(stream)))


def grpo_async_validate_sync(version_ids, token_version, cu_seqlens, group_ids, target_ids,
                             logp_behav, N, T, P, V, G, tbs, v_theta, K, traj_flags, group_count,
                             stale_hist, summary, stream=None, raise_on_invalid=False):
    """Returns (status, summary dict); GRPO_ERR_VALIDATION is returned, not raised, unless asked."""
    host = ValidateSummary()
    status = LIB.grpo_async_validate_sync(
        _ptr(version_ids, torch.int64, "version_ids"), _ptr(token_version, torch.int64, "token_version"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), _ptr(group_ids, torch.int32, "group_ids"),
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(logp_behav, torch.float32, "logp_behav"),
        N, T, P, V, G, tbs, v_theta, K, _ptr(traj_flags, torch.int32, "traj_flags"),
        _ptr(group_count, torch.int32, "group_count"), _ptr(stale_hist, torch.int32, "stale_hist"),
        _ptr(summary, torch.int64, "summary"), C.byref(host), _stream(stream))
    if status != GRPO_OK and (status != GRPO_ERR_VALIDATION or raise_on_invalid):
        _check(status)
    return status, host.as_dict()


def grpo_async_advantage(rewards, group_ids, cu_seqlens, N, P, std_floor, adv, inv_norm,
                         group_count=None, stream=None):
    _check(LIB.grpo_async_advantage(
        _ptr(rewards, torch.float32, "rewards"), _ptr(group_ids, torch.int32, "group_ids"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, P, float(std_floor),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"),
        _ptr(group_count, torch.int32, "group_count"), _stream(stream)))


def _opts(eps_lo, eps_hi, norm, traj_mask, std_unbiased=False):
    return LossOpts(float(eps_lo), float(eps_hi), int(norm),
                    _ptr(traj_mask, torch.uint8, "traj_mask"), int(bool(std_unbiased)))


def grpo_async_advantage_ex(rewards, group_ids, cu_seqlens, N, P, std_floor, eps_lo, eps_hi, norm,
                            traj_mask, adv, inv_norm, group_count=None, stream=None,
                            std_unbiased=False):
    o = _opts(eps_lo, eps_hi, norm, traj_mask, std_unbiased)
    _check(LIB.grpo_async_advantage_ex(
        _ptr(rewards, torch.float32, "rewards"), _ptr(group_ids, torch.int32, "group_ids"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, P, float(std_floor), C.byref(o),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"),
        _ptr(group_count, torch.int32, "group_count"), _stream(stream)))


def _tune(tune):
    if tune is None:
        return None
    return C.byref(Tune(*[int(tune.get(k, 0)) for k in ("kernel", "cluster_size", "ctas_per_sm",
                                                       "stages", "lag", "prefetch", "row_cache", "chunk_kb")]))


def grpo_async_loss_fwd_ex(logits, row_begin, n_rows, V, ld, target_ids, logp_behav, cu_seqlens,
                           N, traj_index, adv, inv_norm, eps_lo, eps_hi, norm, traj_mask,
                           grad_scale, logp_out, lse_out, token_scale_out, traj_sum, stats,
                           dlogits, workspace, tune=None, stream=None):
    for name, x in (("logits", logits), ("dlogits", dlogits)):
        if x is not None and x.element_size() != 2:
            raise TypeError(f"{name}: expected a 16-bit (bf16) tensor")
    o = _opts(eps_lo, eps_hi, norm, traj_mask)
    tp = _tune(tune)
    _check(LIB.grpo_async_loss_fwd_ex(
        _ptr(logits, None, "logits"), row_begin, n_rows, V, ld,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(logp_behav, torch.float32, "logp_behav"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, _ptr(traj_index, torch.int32, "traj_index"),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"), C.byref(o),
        float(grad_scale), _ptr(logp_out, torch.float32, "logp_out"),
        _ptr(lse_out, torch.float32, "lse_out"), _ptr(token_scale_out, torch.float32, "token_scale_out"),
        _ptr(traj_sum, torch.float64, "traj_sum"), _ptr(stats, torch.float64, "stats"),
        _ptr(dlogits, None, "dlogits"), _ptr(workspace, torch.uint8, "workspace"),
        workspace.numel() if workspace is not None else 0, tp, _stream(stream)))


def grpo_async_loss_fwd(logits, row_begin, n_rows, V, ld, target_ids, logp_behav, cu_seqlens, N,
                        traj_index, adv, inv_norm, eps, grad_scale, logp_out, lse_out,
                        token_scale_out, traj_sum, stats, dlogits, workspace, tune=None,
                        stream=None):
    """logits/dlogits: bf16 (or int16/uint16 bit patterns) [n_rows, ld] device tensors."""
    tune_p = None
    if tune is not None:
        t = Tune(*[int(tune.get(k, 0)) for k in ("kernel", "cluster_size", "ctas_per_sm", "stages",
                                                  "lag", "prefetch", "row_cache", "chunk_kb")])
        tune_p = C.byref(t)
    for name, x in (("logits", logits), ("dlogits", dlogits)):
        if x is not None and x.element_size() != 2:
            raise TypeError(f"{name}: expected a 16-bit (bf16) tensor")
    _check(LIB.grpo_async_loss_fwd(
        _ptr(logits, None, "logits"), row_begin, n_rows, V, ld,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(logp_behav, torch.float32, "logp_behav"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, _ptr(traj_index, torch.int32, "traj_index"),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"), float(eps),
        float(grad_scale), _ptr(logp_out, torch.float32, "logp_out"),
        _ptr(lse_out, torch.float32, "lse_out"), _ptr(token_scale_out, torch.float32, "token_scale_out"),
        _ptr(traj_sum, torch.float64, "traj_sum"), _ptr(stats, torch.float64, "stats"),
        _ptr(dlogits, None, "dlogits"), _ptr(workspace, torch.uint8, "workspace"),
        workspace.numel() if workspace is not None else 0, tune_p, _stream(stream)))


def _addr(x, name):
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        return _ptr(x, None, name)
    return int(x)


def grpo_async_loss_fwd_vp(world, rank_begin, shard_cols, slots, logits, dlogits, xbuf, epoch,
                           row_begin, n_rows, V, ld, target_ids, logp_behav, cu_seqlens, N,
                           traj_index, adv, inv_norm, eps_lo, eps_hi, norm, traj_mask, grad_scale,
                           logp_out, lse_out, token_scale_out, traj_sum, stats, workspace,
                           stream=None, lag=0, dynamic_rows=0):
    """logits / dlogits: the n_local local shards (bf16 tensors or raw device addresses);
    xbuf: all `world` exchange buffers as seen from this process (peer addresses), each
    2 * slots * world * 32 bytes."""
    n_local = len(logits)
    if len(xbuf) != world or world > VP_MAX_RANKS:
        raise ValueError("xbuf needs one entry per rank, world <= 8")
    dl = list(dlogits) if dlogits is not None else [None] * n_local
    c = VpComm()
    c.world, c.rank_begin, c.n_local, c.shard_cols, c.slots, c.epoch = world, rank_begin, \
        n_local, shard_cols, slots, epoch
    c.lag = int(lag)
    c.dynamic_rows = int(dynamic_rows)
    for i in range(n_local):
        c.logits[i] = _addr(logits[i], "logits")
        c.dlogits[i] = _addr(dl[i], "dlogits")
    for q in range(world):
        c.xbuf[q] = _addr(xbuf[q], "xbuf")
    o = _opts(eps_lo, eps_hi, norm, traj_mask)
    _check(LIB.grpo_async_loss_fwd_vp(
        C.byref(c), row_begin, n_rows, V, ld,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(logp_behav, torch.float32, "logp_behav"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, _ptr(traj_index, torch.int32, "traj_index"),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"), C.byref(o),
        float(grad_scale), _ptr(logp_out, torch.float32, "logp_out"),
        _ptr(lse_out, torch.float32, "lse_out"), _ptr(token_scale_out, torch.float32, "token_scale_out"),
        _ptr(traj_sum, torch.float64, "traj_sum"), _ptr(stats, torch.float64, "stats"),
        _ptr(workspace, torch.uint8, "workspace"),
        workspace.numel() if workspace is not None else 0, _stream(stream)))


def grpo_async_loss_bwd(logits, n_rows, V, ld, target_ids, lse, token_scale, grad_scale_mult,
                        dlogits, stream=None):
    for name, x in (("logits", logits), ("dlogits", dlogits)):
        if x is not None and x.element_size() != 2:
            raise TypeError(f"{name}: expected a 16-bit (bf16) tensor")
    _check(LIB.grpo_async_loss_bwd(
        _ptr(logits, None, "logits"), n_rows, V, ld, _ptr(target_ids, torch.int64, "target_ids"),
        _ptr(lse, torch.float32, "lse"), _ptr(token_scale, torch.float32, "token_scale"),
        float(grad_scale_mult), _ptr(dlogits, None, "dlogits"), _stream(stream)))


# ---- LM-head-fused loss
def _bf16(x, name):
    if x is not None and x.element_size() != 2:
        raise TypeError(f"{name}: expected a 16-bit (bf16) tensor")
    return _ptr(x, None, name)


def grpo_async_lmhead_workspace_size(n_rows: int, V: int, N: int) -> int:
    return int(LIB.grpo_async_lmhead_workspace_size(n_rows, V, N))


def grpo_async_lmhead_fwd(hidden, W, row_begin, n_rows, d, V, target_ids, logp_behav, cu_seqlens,
                          N, traj_index, adv, inv_norm, eps_lo, eps_hi, norm, traj_mask,
                          grad_scale, logp_out, lse_out, token_scale_out, traj_sum, stats,
                          workspace, stream=None):
    o = _opts(eps_lo, eps_hi, norm, traj_mask)
    _check(LIB.grpo_async_lmhead_fwd(
        _bf16(hidden, "hidden"), _bf16(W, "W"), row_begin, n_rows, d, V,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(logp_behav, torch.float32, "logp_behav"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, _ptr(traj_index, torch.int32, "traj_index"),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"), C.byref(o),
        float(grad_scale), _ptr(logp_out, torch.float32, "logp_out"),
        _ptr(lse_out, torch.float32, "lse_out"), _ptr(token_scale_out, torch.float32, "token_scale_out"),
        _ptr(traj_sum, torch.float64, "traj_sum"), _ptr(stats, torch.float64, "stats"),
        _ptr(workspace, torch.uint8, "workspace"),
        workspace.numel() if workspace is not None else 0, _stream(stream)))


def grpo_async_lmhead_bwd(hidden, W, n_rows, d, V, target_ids, lse, token_scale, grad_scale_mult,
                          dz, ld_dz, dhidden, dW, stream=None):
    _check(LIB.grpo_async_lmhead_bwd(
        _bf16(hidden, "hidden"), _bf16(W, "W"), n_rows, d, V,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(lse, torch.float32, "lse"),
        _ptr(token_scale, torch.float32, "token_scale"), float(grad_scale_mult), _bf16(dz, "dz"),
        ld_dz, _bf16(dhidden, "dhidden"), _ptr(dW, torch.float32, "dW"), _stream(stream)))


def grpo_async_lmhead_logits(hidden, W, n_rows, d, V, out, ld_out, stream=None):
    _check(LIB.grpo_async_lmhead_logits(_bf16(hidden, "hidden"), _bf16(W, "W"), n_rows, d, V,
                                        _bf16(out, "out"), ld_out, _stream(stream)))


def grpo_async_lmhead_set_cta_group(cta_group: int) -> None:
    _check(LIB.grpo_async_lmhead_set_cta_group(int(cta_group)))


# ---- sharded rewards: group statistics through the caller's all-reduce
def grpo_async_group_partials(rewards, group_ids, cu_seqlens, N, P, part, traj_mask=None,
                              stream=None):
    o = _opts(0.2, 0.2, NORM_SEQ, traj_mask)
    _check(LIB.grpo_async_group_partials(
        _ptr(rewards, torch.float32, "rewards"), _ptr(group_ids, torch.int32, "group_ids"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, P, C.byref(o),
        _ptr(part, torch.float64, "part"), _stream(stream)))


def grpo_async_group_sq_partials(rewards, group_ids, N, P, glob, ss, stream=None):
    _check(LIB.grpo_async_group_sq_partials(
        _ptr(rewards, torch.float32, "rewards"), _ptr(group_ids, torch.int32, "group_ids"), N, P,
        _ptr(glob, torch.float64, "glob"), _ptr(ss, torch.float64, "ss"), _stream(stream)))


def grpo_async_advantage_from_stats(rewards, group_ids, cu_seqlens, N, P, std_floor, norm,
                                    traj_mask, std_unbiased, glob, ss, adv, inv_norm, stream=None):
    o = _opts(0.2, 0.2, norm, traj_mask, std_unbiased)
    _check(LIB.grpo_async_advantage_from_stats(
        _ptr(rewards, torch.float32, "rewards"), _ptr(group_ids, torch.int32, "group_ids"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, P, float(std_floor), C.byref(o),
        _ptr(glob, torch.float64, "glob"), _ptr(ss, torch.float64, "ss"),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"), _stream(stream)))


# ---- tensor-parallel LM head (NEXT(2) x NEXT(3))
def grpo_async_lmhead_tp_partials(hidden, W_shard, n_rows, d, Vs, col_offset, target_ids, row_part,
                                  workspace, stream=None):
    _check(LIB.grpo_async_lmhead_tp_partials(
        _bf16(hidden, "hidden"), _bf16(W_shard, "W_shard"), n_rows, d, Vs, col_offset,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(row_part, torch.float32, "row_part"),
        _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream)))


def grpo_async_lmhead_tp_fwd(row_parts, R, row_begin, n_rows, V, target_ids, logp_behav,
                             cu_seqlens, N, traj_index, adv, inv_norm, eps_lo, eps_hi, norm,
                             traj_mask, grad_scale, logp_out, lse_out, token_scale_out, traj_sum,
                             stats, workspace, stream=None):
    o = _opts(eps_lo, eps_hi, norm, traj_mask)
    _check(LIB.grpo_async_lmhead_tp_fwd(
        _ptr(row_parts, torch.float32, "row_parts"), R, row_begin, n_rows, V,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(logp_behav, torch.float32, "logp_behav"),
        _ptr(cu_seqlens, torch.int64, "cu_seqlens"), N, _ptr(traj_index, torch.int32, "traj_index"),
        _ptr(adv, torch.float32, "adv"), _ptr(inv_norm, torch.float32, "inv_norm"), C.byref(o),
        float(grad_scale), _ptr(logp_out, torch.float32, "logp_out"),
        _ptr(lse_out, torch.float32, "lse_out"), _ptr(token_scale_out, torch.float32, "token_scale_out"),
        _ptr(traj_sum, torch.float64, "traj_sum"), _ptr(stats, torch.float64, "stats"),
        _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream)))


def grpo_async_lmhead_tp_bwd(hidden, W_shard, n_rows, d, Vs, col_offset, target_ids, lse,
                             token_scale, grad_scale_mult, dz, ld_dz, dhidden_partial, dW_shard,
                             stream=None):
    _check(LIB.grpo_async_lmhead_tp_bwd(
        _bf16(hidden, "hidden"), _bf16(W_shard, "W_shard"), n_rows, d, Vs, col_offset,
        _ptr(target_ids, torch.int64, "target_ids"), _ptr(lse, torch.float32, "lse"),
        _ptr(token_scale, torch.float32, "token_scale"), float(grad_scale_mult), _bf16(dz, "dz"),
        ld_dz, _ptr(dhidden_partial, torch.float32, "dhidden_partial"),
        _ptr(dW_shard, torch.float32, "dW_shard"), _stream(stream)))


def grpo_async_lmhead_dw(hidden, n_rows, d, V, dz, ld_dz, dW, stream=None):
    _check(LIB.grpo_async_lmhead_dw(_bf16(hidden, "hidden"), n_rows, d, V, _bf16(dz, "dz"), ld_dz,
                                    _ptr(dW, torch.float32, "dW"), _stream(stream)))


def grpo_async_lmhead_dx(dz, ld_dz, W, n_rows, d, V, dhidden, stream=None):
    """dhidden = dz W on the tensor cores (bf16 or float32 [n_rows, d] by dhidden's dtype)."""
    out_bf16 = 1 if dhidden.element_size() == 2 else 0
    _check(LIB.grpo_async_lmhead_dx(_bf16(dz, "dz"), ld_dz, _bf16(W, "W"), n_rows, d, V,
                                    _ptr(dhidden, None, "dhidden"), out_bf16, _stream(stream)))


def grpo_async_lmhead_tp_dx(dz, ld_dz, W_shard, n_rows, d, Vs, world, rank, slots, epoch=0,
                            stream=None):
    """slots: `world` device addresses (ints or float32 tensors) of every rank's slot buffer
    ([2][world][rows_per_rank][d] f32; call `epoch` writes half epoch % 2)."""
    arr = (C.c_void_p * world)(*[_addr(x, "slots") for x in slots])
    _check(LIB.grpo_async_lmhead_tp_dx(_bf16(dz, "dz"), ld_dz, _bf16(W_shard, "W_shard"), n_rows, d,
                                       Vs, world, rank, arr, epoch, _stream(stream)))


def grpo_async_lmhead_tp_dx_reduce(own_slots, world, n_rows, d, rank, out, epoch=0, stream=None):
    out_bf16 = 1 if out.element_size() == 2 else 0
    _check(LIB.grpo_async_lmhead_tp_dx_reduce(_ptr(own_slots, torch.float32, "own_slots"), world,
                                              n_rows, d, rank, _ptr(out, None, "out"), out_bf16,
                                              epoch, _stream(stream)))
