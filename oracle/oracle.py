"""oracle/oracle.py -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes binding to the plain fp64 C oracle in ``oracle/grpo_oracle.c``
(arxiv 2604.26256, PAPER.md eq:grpo_async P:9-26, eq:ratio_async P:28-40,
eq:group_advantage P:153-156), plus the LM-head composition of SURVEY NEXT(2)
(logits = X W^T in fp64, pinned by the one-hot and finite-difference tests).  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` leg may import this module.
It never imports the CUDA package and the CUDA package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "grpo_oracle.c")
LIB = os.path.join(HERE, "libgrpo_oracle.so")

FLAG_NAMES = ["STALE", "FUTURE", "ZERO_LEN", "BAD_GROUP_ID", "GROUP_SIZE",
              "C1_MIXED", "BAD_TARGET", "BAD_LOGP_BEHAV"]


class ValidateSummary(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_traj", "n_tokens", "n_stale", "n_future", "n_zero_len",
        "n_bad_group_id", "n_group_size", "n_c1_mixed", "n_bad_target",
        "n_bad_logp_behav", "n_groups_wrong_size", "c2_dropped",
        "max_staleness", "min_staleness", "cu_ok", "tbs_ok", "c1_ok", "c2_ok",
        "c3_ok", "valid")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile the oracle with the flags its header states (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off",
                               "-fopenmp", "-shared", "-fPIC", "-std=c11", "-Wall",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i32, i64, f32, f64 = C.c_int32, C.c_int64, C.c_float, C.c_double
        _lib.oracle_validate.argtypes = [i32, i64, i32, i32, i32, i32, i64, i32,
                                         P, P, P, P, P, P, P, P, P, P]
        _lib.oracle_validate.restype = C.c_int
        _lib.oracle_advantage.argtypes = [i32, i32, P, P, P, f64, P, P, P]
        _lib.oracle_advantage.restype = None
        _lib.oracle_advantage_ex.argtypes = [i32, i32, P, P, P, f64, i32, P, P, P]
        _lib.oracle_advantage_ex.restype = None
        _lib.oracle_log_softmax_row.argtypes = [i32, P, i64, P, P]
        _lib.oracle_log_softmax_row.restype = None
        _lib.oracle_token.argtypes = [f64, f32, f64, f64, f32, f64, P, P, P, P]
        _lib.oracle_token.restype = None
        _lib.oracle_dlogits_row.argtypes = [i32, P, i64, f64, f64, P]
        _lib.oracle_dlogits_row.restype = None
        _lib.oracle_rows.argtypes = [i64, P, i32, i64, P, P, P, i32, P, P, P, f32, f64,
                                     P, P, P, P, P, P, P]
        _lib.oracle_rows.restype = None
        _lib.oracle_rows_f64.argtypes = [i64, P, i32, P, P, P, i32, P, P, P, f32, f32, f64,
                                         P, P, P, P, P, P, P]
        _lib.oracle_rows2.argtypes = [i64, P, i32, i64, P, P, P, i32, P, P, P, f32, f32, f64,
                                      P, P, P, P, P, P, P]
        _lib.oracle_rows2.restype = None
        _lib.oracle_token_asym.argtypes = [f64, f32, f64, f64, f32, f32, f64, P, P, P, P]
        _lib.oracle_token_asym.restype = None
        _lib.oracle_weights.argtypes = [i32, i32, P, P, P, i32, P, P]
        _lib.oracle_weights.restype = None
        _lib.oracle_rows_f64.restype = None
        _lib.oracle_objective_tokens.argtypes = [i32, P, P, P, P]
        _lib.oracle_objective_tokens.restype = f64
        _lib.oracle_objective_nested.argtypes = [i32, i32, P, P, P, P]
        _lib.oracle_objective_nested.restype = f64
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------- O1
def validate(version_ids, cu_seqlens, group_ids, target_ids, *, P, V, G, tbs,
             v_theta, K, token_version=None, logp_behav=None):
    version_ids = _c(version_ids, np.int64)
    cu = _c(cu_seqlens, np.int64)
    gids = _c(group_ids, np.int32)
    tgt = _c(target_ids, np.int64)
    tv = _c(token_version, np.int64)
    lw = _c(logp_behav, np.float32)
    N = len(version_ids)
    T = len(tgt)
    flags = np.zeros(N, np.uint32)
    gc = np.zeros(max(P, 1), np.int32)
    hist = np.zeros(max(P * (K + 1), 1), np.int32)
    summ = ValidateSummary()
    rc = lib().oracle_validate(N, T, P, V, G, tbs, v_theta, K, _p(version_ids), _p(tv),
                               _p(cu), _p(gids), _p(tgt), _p(lw), _p(flags), _p(gc),
                               _p(hist), C.byref(summ))
    return dict(rc=rc, traj_flags=flags, group_count=gc[:P],
                stale_hist=hist[:P * (K + 1)].reshape(P, K + 1), summary=summ.as_dict())


# --------------------------------------------------------------------------- O2
def advantage(rewards, group_ids, cu_seqlens, P, std_floor=1e-8, unbiased=False):
    """eq:group_advantage; unbiased=True: sample std (n - 1), SURVEY NEXT(1)."""
    R = _c(rewards, np.float32)
    g = _c(group_ids, np.int32)
    cu = _c(cu_seqlens, np.int64)
    N = len(R)
    adv = np.zeros(N, np.float64)
    inv = np.zeros(N, np.float64)
    gc = np.zeros(max(P, 1), np.int32)
    lib().oracle_advantage_ex(N, P, _p(R), _p(g), _p(cu), float(std_floor), int(bool(unbiased)),
                              _p(adv), _p(inv), _p(gc))
    return adv, inv, gc[:P]


# --------------------------------------------------------------------------- O3
def log_softmax_row(row_bf16_bits, y):
    row = _c(row_bf16_bits, np.uint16)
    lse = C.c_double()
    logp = C.c_double()
    lib().oracle_log_softmax_row(len(row), _p(row), int(y), C.byref(lse), C.byref(logp))
    return lse.value, logp.value


# --------------------------------------------------------------------------- O4
def token(logp, logp_behav, A, inv_norm, eps, grad_scale=1.0, eps_hi=None):
    r, term, s = C.c_double(), C.c_double(), C.c_double()
    clipped = C.c_int32()
    if eps_hi is None:
        lib().oracle_token(float(logp), float(logp_behav), float(A), float(inv_norm), float(eps),
                           float(grad_scale), C.byref(r), C.byref(term), C.byref(clipped),
                           C.byref(s))
    else:
        lib().oracle_token_asym(float(logp), float(logp_behav), float(A), float(inv_norm),
                                float(eps), float(eps_hi), float(grad_scale), C.byref(r),
                                C.byref(term), C.byref(clipped), C.byref(s))
    return r.value, term.value, bool(clipped.value), s.value


def weights(group_ids, cu_seqlens, group_count, P, norm=0, traj_mask=None):
    """Token weights w_i under the sequence-mean (0) or token-mean (1) normalisation."""
    g = _c(group_ids, np.int32)
    cu = _c(cu_seqlens, np.int64)
    gc = _c(group_count, np.int32)
    m = _c(traj_mask, np.uint8)
    w = np.zeros(len(g), np.float64)
    lib().oracle_weights(len(g), P, _p(g), _p(cu), _p(gc), int(norm), _p(m), _p(w))
    return w


# --------------------------------------------------------------------------- O5
def dlogits_row(row_bf16_bits, y, lse, s):
    row = _c(row_bf16_bits, np.uint16)
    out = np.zeros(len(row), np.float64)
    lib().oracle_dlogits_row(len(row), _p(row), int(y), float(lse), float(s), _p(out))
    return out


@dataclass
class RowsResult:
    lse: np.ndarray
    logp: np.ndarray
    r: np.ndarray
    term: np.ndarray
    clipped: np.ndarray
    s: np.ndarray
    dlogits: np.ndarray | None


def rows(row_ids, logits_bits, V, target_ids, logp_behav, cu_seqlens, adv, inv_norm,
         eps, grad_scale=1.0, want_dlogits=True, eps_hi=None):
    """O3-O5 on a set of global rows.  logits_bits: uint16 [n_rows, ld] (ld >= V).
    eps is the lower clip range; eps_hi (default eps) the upper one."""
    row_ids = _c(row_ids, np.int64)
    lg = np.ascontiguousarray(logits_bits, dtype=np.uint16)
    n = len(row_ids)
    ld = lg.shape[1] if n else V
    tgt = _c(target_ids, np.int64)
    lw = _c(logp_behav, np.float32)
    cu = _c(cu_seqlens, np.int64)
    adv = _c(adv, np.float64)
    inv = _c(inv_norm, np.float64)
    out = {k: np.zeros(n, np.float64) for k in ("lse", "logp", "r", "term", "s")}
    clipped = np.zeros(n, np.int32)
    dl = np.zeros((n, V), np.float64) if want_dlogits else None
    lib().oracle_rows2(n, _p(row_ids), V, ld, _p(lg), _p(tgt), _p(lw), len(adv), _p(cu),
                       _p(adv), _p(inv), float(eps), float(eps if eps_hi is None else eps_hi),
                       float(grad_scale), _p(out["lse"]),
                      _p(out["logp"]), _p(out["r"]), _p(out["term"]), _p(clipped),
                      _p(out["s"]), _p(dl))
    return RowsResult(out["lse"], out["logp"], out["r"], out["term"], clipped.astype(bool),
                      out["s"], dl)


def rows_f64(row_ids, logits_f64, target_ids, logp_behav, cu_seqlens, adv, inv_norm, eps,
             grad_scale=1.0, want_dlogits=True, eps_hi=None):
    """O3-O5 on fp64 logits [n_rows, V] (finite-difference pins)."""
    row_ids = _c(row_ids, np.int64)
    lg = np.ascontiguousarray(logits_f64, dtype=np.float64)
    n, V = lg.shape
    tgt = _c(target_ids, np.int64)
    lw = _c(logp_behav, np.float32)
    cu = _c(cu_seqlens, np.int64)
    adv = _c(adv, np.float64)
    inv = _c(inv_norm, np.float64)
    out = {k: np.zeros(n, np.float64) for k in ("lse", "logp", "r", "term", "s")}
    clipped = np.zeros(n, np.int32)
    dl = np.zeros((n, V), np.float64) if want_dlogits else None
    lib().oracle_rows_f64(n, _p(row_ids), V, _p(lg), _p(tgt), _p(lw), len(adv), _p(cu),
                          _p(adv), _p(inv), float(eps), float(eps if eps_hi is None else eps_hi),
                          float(grad_scale), _p(out["lse"]),
                          _p(out["logp"]), _p(out["r"]), _p(out["term"]), _p(clipped),
                          _p(out["s"]), _p(dl))
    return RowsResult(out["lse"], out["logp"], out["r"], out["term"], clipped.astype(bool),
                      out["s"], dl)


def objective_tokens(cu_seqlens, inv_norm, term):
    cu = _c(cu_seqlens, np.int64)
    inv = _c(inv_norm, np.float64)
    tm = _c(term, np.float64)
    N = len(cu) - 1
    ts = np.zeros(N, np.float64)
    J = lib().oracle_objective_tokens(N, _p(cu), _p(inv), _p(tm), _p(ts))
    return J, ts


def objective_nested(cu_seqlens, group_ids, version_ids, term, P):
    cu = _c(cu_seqlens, np.int64)
    g = _c(group_ids, np.int32)
    v = _c(version_ids, np.int64)
    tm = _c(term, np.float64)
    return lib().oracle_objective_nested(len(cu) - 1, P, _p(cu), _p(g), _p(v), _p(tm))


# --------------------------------------------------------------------- full path
def run_batch(batch, logits_bits, eps=0.2, grad_scale=1.0, std_floor=1e-8, want_dlogits=True,
              eps_hi=None, norm=0, traj_mask=None, std_unbiased=False):
    """Whole hot path on a small batch: validate, advantage, rows, J.

    ``batch`` is a synth.gen.Batch (or anything with the same fields);
    ``logits_bits`` the uint16 [T, ld] bf16 bit patterns of every row.
    """
    val = validate(batch.version_ids, batch.cu_seqlens, batch.group_ids, batch.target_ids,
                   P=batch.P, V=batch.V, G=batch.G, tbs=batch.tbs, v_theta=batch.v_theta,
                   K=batch.K, token_version=batch.token_version, logp_behav=batch.logp_behav)
    adv, inv, gc = advantage(batch.rewards, batch.group_ids, batch.cu_seqlens, batch.P, std_floor,
                             unbiased=std_unbiased)
    if norm != 0 or traj_mask is not None:
        inv = weights(batch.group_ids, batch.cu_seqlens, gc, batch.P, norm, traj_mask)
    T = int(batch.cu_seqlens[-1])
    rr = rows(np.arange(T, dtype=np.int64), logits_bits, batch.V, batch.target_ids,
              batch.logp_behav, batch.cu_seqlens, adv, inv, eps, grad_scale, want_dlogits,
              eps_hi=eps_hi)
    J, traj_sum = objective_tokens(batch.cu_seqlens, inv, rr.term)
    return dict(validate=val, adv=adv, inv_norm=inv, group_count=gc, rows=rr, J=J,
                loss=-J, traj_sum=traj_sum,
                n_clipped=int(rr.clipped.sum()),
                n_active=int(((~rr.clipped) & (adv[_traj_index(batch.cu_seqlens)] != 0)
                              & (inv[_traj_index(batch.cu_seqlens)] != 0)).sum()))


def _traj_index(cu_seqlens):
    cu = np.asarray(cu_seqlens, np.int64)
    return np.repeat(np.arange(len(cu) - 1), np.diff(cu))


# ------------------------------------------------------- NEXT(2): LM-head-fused loss
def _bf16_to_f64(bits):
    """bf16 bit patterns -> float64 (exact: a bf16 is a float32 with 16 zero low bits)."""
    b = np.ascontiguousarray(bits, np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def lmhead_logits(hidden_bits, W_bits):
    """z = X W^T (the trainer's LM head) in fp64 from bf16 X [n, d] and W [V, d].
    Every product of two bf16 values is exact in fp64; the library matmul is the step."""
    return _bf16_to_f64(hidden_bits) @ _bf16_to_f64(W_bits).T


def run_batch_lmhead(batch, hidden_bits, W_bits, eps=0.2, grad_scale=1.0, std_floor=1e-8,
                     want_grads=True, eps_hi=None, norm=0, traj_mask=None, std_unbiased=False):
    """The whole path with logits = X W^T: validate, advantage, O3-O5 on
    the fp64 logits, J; with want_grads the chain rule through the LM head:
      dz = dJ/dz (O5 rows), dJ/dX = dz W, dJ/dW = dz^T X."""
    val = validate(batch.version_ids, batch.cu_seqlens, batch.group_ids, batch.target_ids,
                   P=batch.P, V=batch.V, G=batch.G, tbs=batch.tbs, v_theta=batch.v_theta,
                   K=batch.K, token_version=batch.token_version, logp_behav=batch.logp_behav)
    adv, inv, gc = advantage(batch.rewards, batch.group_ids, batch.cu_seqlens, batch.P, std_floor,
                             unbiased=std_unbiased)
    if norm != 0 or traj_mask is not None:
        inv = weights(batch.group_ids, batch.cu_seqlens, gc, batch.P, norm, traj_mask)
    T = int(batch.cu_seqlens[-1])
    z = lmhead_logits(hidden_bits, W_bits)
    rr = rows_f64(np.arange(T, dtype=np.int64), z, batch.target_ids, batch.logp_behav,
                  batch.cu_seqlens, adv, inv, eps, grad_scale, want_grads, eps_hi=eps_hi)
    J, traj_sum = objective_tokens(batch.cu_seqlens, inv, rr.term)
    out = dict(validate=val, adv=adv, inv_norm=inv, group_count=gc, rows=rr, J=J, loss=-J,
               traj_sum=traj_sum, logits=z, n_clipped=int(rr.clipped.sum()))
    if want_grads:
        out["dhidden"] = rr.dlogits @ _bf16_to_f64(W_bits)
        out["dW"] = rr.dlogits.T @ _bf16_to_f64(hidden_bits)
    return out


def lmhead_logits_rows(hidden_rows_bits, W_bits, block=16384):
    """lmhead_logits for a few rows of X against a large W, W widened block by block (the same
    definition, bounded memory: full-size parity tests)."""
    Xr = _bf16_to_f64(hidden_rows_bits)
    V = W_bits.shape[0]
    out = np.empty((Xr.shape[0], V), np.float64)
    for v0 in range(0, V, block):
        out[:, v0:v0 + block] = Xr @ _bf16_to_f64(W_bits[v0:v0 + block]).T
    return out


def matmul_rows_W(rows_f64, W_bits, block=16384):
    """rows [k, V] (fp64) times W [V, d] (bf16, widened block by block): dJ/dX of the rows."""
    V, d = W_bits.shape
    out = np.zeros((rows_f64.shape[0], d), np.float64)
    for v0 in range(0, V, block):
        out += rows_f64[:, v0:v0 + block] @ _bf16_to_f64(W_bits[v0:v0 + block])
    return out
