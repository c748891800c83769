"""Thin ctypes binding of include/grpo_transfer_queue.h: the host control plane
(sliding version window + TransferQueue) that forms the
group-atomic, staleness-bounded batches the loss consumes.  Marshalling only."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

_lib = L.LIB
_P, _i32, _i64, _f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
_lib.grpo_tq_create.argtypes = [_i32, _i32, _i64]
_lib.grpo_tq_create.restype = _P
_lib.grpo_tq_destroy.argtypes = [_P]
_lib.grpo_tq_destroy.restype = None
_lib.grpo_tq_dispatch.argtypes = [_P, _i64, _i32]
_lib.grpo_tq_dispatch.restype = C.c_int
_lib.grpo_tq_push.argtypes = [_P, _i64, _i64, _i64, _i64, _f32]
_lib.grpo_tq_push.restype = C.c_int
_lib.grpo_tq_form_batch.argtypes = [_P, _i32, _i64, _P, _P, _P, _P, _P, _P, _P]
_lib.grpo_tq_form_batch.restype = C.c_int
_lib.grpo_tq_advance.argtypes = [_P, _i64, _P, _P, _P]
_lib.grpo_tq_advance.restype = C.c_int
_lib.grpo_tq_stats.argtypes = [_P, _P, _P]
_lib.grpo_tq_stats.restype = C.c_int

EXPORTED = ("grpo_tq_create", "grpo_tq_destroy", "grpo_tq_dispatch", "grpo_tq_push",
            "grpo_tq_form_batch", "grpo_tq_advance", "grpo_tq_stats")


class TqStats(C.Structure):
    _fields_ = [("newest", _i64), ("oldest", _i64), ("window_size", _i32), ("queued", _i64),
                ("in_flight", _i64), ("pushed", _i64), ("consumed", _i64), ("batches", _i64),
                ("max_staleness", _i64)]


@dataclass
class FormedBatch:
    request_ids: np.ndarray
    prompt_ids: np.ndarray
    group_ids: np.ndarray
    version_ids: np.ndarray
    lengths: np.ndarray
    rewards: np.ndarray

    @property
    def cu_seqlens(self):
        cu = np.zeros(len(self.lengths) + 1, np.int64)
        cu[1:] = np.cumsum(self.lengths)
        return cu


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class TransferQueue:
    def __init__(self, G: int, K: int, first_version: int):
        self.h = _lib.grpo_tq_create(G, K, first_version)
        if not self.h:
            raise ValueError(f"grpo_tq_create(G={G}, K={K}) failed")
        self.G, self.K = G, K

    def __del__(self):
        if getattr(self, "h", None):
            _lib.grpo_tq_destroy(self.h)
            self.h = None

    def dispatch(self, version: int, n: int):
        L._check(_lib.grpo_tq_dispatch(self.h, version, n))

    def push(self, request_id: int, prompt_id: int, version: int, length: int, reward: float):
        L._check(_lib.grpo_tq_push(self.h, request_id, prompt_id, version, length, reward))

    def form_batch(self, tbs: int, v_theta: int):
        out = dict(request_ids=np.zeros(max(tbs, 1), np.int64),
                   prompt_ids=np.zeros(max(tbs, 1), np.int64),
                   group_ids=np.zeros(max(tbs, 1), np.int32),
                   version_ids=np.zeros(max(tbs, 1), np.int64),
                   lengths=np.zeros(max(tbs, 1), np.int64), rewards=np.zeros(max(tbs, 1), np.float32))
        formed = C.c_int32()
        L._check(_lib.grpo_tq_form_batch(self.h, tbs, v_theta, C.byref(formed),
                                         _ptr(out["request_ids"]), _ptr(out["prompt_ids"]),
                                         _ptr(out["group_ids"]), _ptr(out["version_ids"]),
                                         _ptr(out["lengths"]), _ptr(out["rewards"])))
        if not formed.value:
            return None
        return FormedBatch(**{k: v[:tbs] for k, v in out.items()})

    def advance(self, new_version: int):
        adv, rin, rq = C.c_int32(), C.c_int64(), C.c_int64()
        L._check(_lib.grpo_tq_advance(self.h, new_version, C.byref(adv), C.byref(rin), C.byref(rq)))
        return bool(adv.value), int(rin.value), int(rq.value)

    def stats(self):
        st = TqStats()
        vers = np.zeros(self.K, np.int64)
        L._check(_lib.grpo_tq_stats(self.h, C.byref(st), _ptr(vers)))
        d = {n: int(getattr(st, n)) for n, _ in TqStats._fields_}
        d["window"] = vers[:d["window_size"]].tolist()
        return d
