"""-m "not gpu": the C-ABI library loads and exports every symbol include/grpo_async.h
declares; host-side argument checks return their documented status codes without
touching the GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("grpo_async.h", "grpo_transfer_queue.h")]


def declared_functions():
    src = "\n".join(open(h).read() for h in HEADERS)
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(grpo_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("grpo_async_advantage", "grpo_async_loss_fwd", "grpo_async_loss_bwd",
              "grpo_async_validate"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2604_26256_b200._lib as L
    lib = C.CDLL(L.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    import paper_2604_26256_b200.transfer_queue as TQ
    assert set(L.EXPORTED) | set(TQ.EXPORTED) == set(declared_functions())


def test_binding_names_match_c_entry_points():
    import paper_2604_26256_b200 as G
    for n in declared_functions():
        if not n.startswith("grpo_tq_"):
            assert hasattr(G._lib, n), n


def test_host_side_errors_without_gpu():
    """Argument errors are detected on the host before any CUDA call."""
    import paper_2604_26256_b200._lib as L
    lib = L.LIB
    ws = L.LIB.grpo_async_workspace_size(100, 1000, 4)
    assert ws >= 100 * 16
    fake = C.c_void_p(16)  # never dereferenced: every call below fails its host checks first
    # N <= 0
    st = lib.grpo_async_loss_fwd(fake, 0, 10, 1000, 1000, fake, fake, fake, 0, None, fake, fake,
                                 0.2, 1.0, None, None, None, fake, fake, None, fake, ws, None, None)
    assert st == L.GRPO_ERR_INVALID_ARG and b"N=0" in lib.grpo_last_error()
    # eps out of range
    st = lib.grpo_async_loss_fwd(fake, 0, 10, 1000, 1000, fake, fake, fake, 4, None, fake, fake,
                                 1.5, 1.0, None, None, None, fake, fake, None, fake, ws, None, None)
    assert st == L.GRPO_ERR_INVALID_ARG
    # ld % 8 != 0 and ld < V
    for ld in (1001, 999):
        st = lib.grpo_async_loss_fwd(fake, 0, 10, 1000, ld, fake, fake, fake, 4, None, fake, fake,
                                     0.2, 1.0, None, None, None, fake, fake, None, fake, ws, None,
                                     None)
        assert st == L.GRPO_ERR_ALIGNMENT
    # misaligned logits pointer
    st = lib.grpo_async_loss_fwd(C.c_void_p(18), 0, 10, 1000, 1000, fake, fake, fake, 4, None, fake,
                                 fake, 0.2, 1.0, None, None, None, fake, fake, None, fake, ws, None,
                                 None)
    assert st == L.GRPO_ERR_ALIGNMENT
    # workspace too small
    st = lib.grpo_async_loss_fwd(fake, 0, 10, 1000, 1000, fake, fake, fake, 4, None, fake, fake,
                                 0.2, 1.0, None, None, None, fake, fake, None, fake, 8, None, None)
    assert st == L.GRPO_ERR_WORKSPACE
    # advantage: std_floor <= 0, P <= 0
    assert lib.grpo_async_advantage(fake, fake, fake, 4, 1, 0.0, fake, fake, None,
                                    None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_advantage(fake, fake, fake, 4, 0, 1e-8, fake, fake, None,
                                    None) == L.GRPO_ERR_INVALID_ARG
    # validate: K < 0, NULL summary
    assert lib.grpo_async_validate(fake, None, fake, fake, fake, None, 4, 10, 1, 100, 4, 4, 1000,
                                   -1, fake, fake, fake, fake, None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_validate(fake, None, fake, fake, fake, None, 4, 10, 1, 100, 4, 4, 1000,
                                   1, fake, fake, fake, None, None) == L.GRPO_ERR_INVALID_ARG
    # loss_bwd: NULL lse
    assert lib.grpo_async_loss_bwd(fake, 10, 100, 104, fake, None, fake, 1.0, fake,
                                   None) == L.GRPO_ERR_INVALID_ARG
    # profile collect with NULL outputs
    assert lib.grpo_profile_collect(None, None) == L.GRPO_ERR_INVALID_ARG


def test_package_has_no_cpu_fallback():
    """The product package never imports the oracle; the binding only marshals."""
    pkg = os.path.join(ROOT, "paper_2604_26256_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("oracle/", "").lower() or fn == "build.py", fn


def test_host_side_errors_new_entry_points():
    """NEXT(2) / NEXT(3) / K3c entry points: documented status codes on bad arguments,
    returned by the host checks before any CUDA call."""
    import paper_2604_26256_b200._lib as L
    lib = L.LIB
    fake = C.c_void_p(16)
    ws = lib.grpo_async_lmhead_workspace_size(100, 1000, 4)
    assert ws >= lib.grpo_async_workspace_size(100, 1000, 4)
    opts = L.LossOpts(0.2, 0.2, 0, None, 0)
    # LM head: d not a multiple of 64, misaligned W, workspace too small, NULL opts
    st = lib.grpo_async_lmhead_fwd(fake, fake, 0, 10, 96, 1000, fake, fake, fake, 4, None, fake,
                                   fake, C.byref(opts), 1.0, None, None, None, fake, fake, fake, ws,
                                   None)
    assert st == L.GRPO_ERR_INVALID_ARG and b"multiple of 64" in lib.grpo_last_error()
    st = lib.grpo_async_lmhead_fwd(fake, C.c_void_p(18), 0, 10, 128, 1000, fake, fake, fake, 4, None,
                                   fake, fake, C.byref(opts), 1.0, None, None, None, fake, fake, fake,
                                   ws, None)
    assert st == L.GRPO_ERR_ALIGNMENT
    st = lib.grpo_async_lmhead_fwd(fake, fake, 0, 10, 128, 1000, fake, fake, fake, 4, None, fake,
                                   fake, C.byref(opts), 1.0, None, None, None, fake, fake, fake, 8,
                                   None)
    assert st == L.GRPO_ERR_WORKSPACE
    st = lib.grpo_async_lmhead_fwd(fake, fake, 0, 10, 128, 1000, fake, fake, fake, 4, None, fake,
                                   fake, None, 1.0, None, None, None, fake, fake, fake, ws, None)
    assert st == L.GRPO_ERR_INVALID_ARG
    # LM-head backward: ld_dz < V; logits: ld_out not a multiple of 8
    st = lib.grpo_async_lmhead_bwd(fake, fake, 10, 128, 1000, fake, fake, fake, 1.0, fake, 999,
                                   None, None, None)
    assert st == L.GRPO_ERR_ALIGNMENT
    st = lib.grpo_async_lmhead_logits(fake, fake, 10, 128, 1000, fake, 1004, None)
    assert st == L.GRPO_ERR_ALIGNMENT
    # vocabulary-parallel: world > 8, shard_cols % 8, shards that do not cover V, slots < n_rows
    c = L.VpComm()
    c.world, c.rank_begin, c.n_local, c.shard_cols, c.slots = 9, 0, 1, 128, 100
    vws = lib.grpo_async_workspace_size(10, 1000, 4)
    args = lambda: (C.byref(c), 0, 10, 1000, 1024, fake, fake, fake, 4, None, fake, fake,
                    C.byref(opts), 1.0, None, None, None, fake, fake, fake, vws, None)
    assert lib.grpo_async_loss_fwd_vp(*args()) == L.GRPO_ERR_INVALID_ARG
    c.world, c.shard_cols = 2, 500
    assert lib.grpo_async_loss_fwd_vp(*args()) == L.GRPO_ERR_INVALID_ARG
    c.shard_cols = 256
    assert lib.grpo_async_loss_fwd_vp(*args()) == L.GRPO_ERR_INVALID_ARG   # 2 * 256 < V
    c.shard_cols, c.slots = 504, 5
    assert lib.grpo_async_loss_fwd_vp(*args()) == L.GRPO_ERR_INVALID_ARG   # slots < n_rows
    # tune: kernel out of range
    t = L.Tune(4, 0, 0, 0, 0, 0, 0, 0)
    ws2 = lib.grpo_async_workspace_size(10, 1000, 4)
    st = lib.grpo_async_loss_fwd(fake, 0, 10, 1000, 1000, fake, fake, fake, 4, None, fake, fake,
                                 0.2, 1.0, None, None, None, fake, fake, None, fake, ws2,
                                 C.byref(t), None)
    assert st == L.GRPO_ERR_INVALID_ARG


def test_host_side_errors_tensor_parallel_and_sharded_entry_points():
    import paper_2604_26256_b200._lib as L
    lib = L.LIB
    fake = C.c_void_p(16)
    assert lib.grpo_async_lmhead_set_cta_group(3) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_lmhead_set_cta_group(2) == L.GRPO_OK
    ws = lib.grpo_async_lmhead_workspace_size(10, 1000, 1)
    # tp partials: negative col_offset, d % 64
    assert lib.grpo_async_lmhead_tp_partials(fake, fake, 10, 128, 1000, -1, fake, fake, fake, ws,
                                             None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_lmhead_tp_partials(fake, fake, 10, 100, 1000, 0, fake, fake, fake, ws,
                                             None) == L.GRPO_ERR_INVALID_ARG
    # tp fwd: R < 1, NULL opts
    opts = L.LossOpts(0.2, 0.2, 0, None, 0)
    vws = lib.grpo_async_workspace_size(10, 1000, 4)
    assert lib.grpo_async_lmhead_tp_fwd(fake, 0, 0, 10, 1000, fake, fake, fake, 4, None, fake, fake,
                                        C.byref(opts), 1.0, None, None, None, fake, fake, fake, vws,
                                        None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_lmhead_tp_fwd(fake, 2, 0, 10, 1000, fake, fake, fake, 4, None, fake, fake,
                                        None, 1.0, None, None, None, fake, fake, fake, vws,
                                        None) == L.GRPO_ERR_INVALID_ARG
    # tp bwd: ld_dz < Vs
    assert lib.grpo_async_lmhead_tp_bwd(fake, fake, 10, 128, 1000, 0, fake, fake, fake, 1.0, fake, 992,
                                        None, None, None) == L.GRPO_ERR_ALIGNMENT
    # fused dhidden: d % 128, rank >= world, NULL slot
    slots = (C.c_void_p * 2)(16, 32)
    assert lib.grpo_async_lmhead_tp_dx(fake, 1000, fake, 10, 192, 1000, 2, 0, slots, 0,
                                       None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_lmhead_tp_dx(fake, 1000, fake, 10, 256, 1000, 2, 2, slots, 0,
                                       None) == L.GRPO_ERR_INVALID_ARG
    bad = (C.c_void_p * 2)(16, None)
    assert lib.grpo_async_lmhead_tp_dx(fake, 1000, fake, 10, 256, 1000, 2, 0, bad, 1,
                                       None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_lmhead_tp_dx_reduce(fake, 9, 10, 256, 0, fake, 0, 0, None) == L.GRPO_ERR_INVALID_ARG
    # dW from dz: ld_dz not a multiple of 8
    assert lib.grpo_async_lmhead_dw(fake, 10, 128, 1000, fake, 1001, fake, None) == L.GRPO_ERR_ALIGNMENT
    # sharded rewards: P <= 0, std_floor <= 0
    assert lib.grpo_async_group_partials(fake, fake, fake, 4, 0, None, fake, None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_group_sq_partials(fake, fake, 4, 2, None, fake, None) == L.GRPO_ERR_INVALID_ARG
    assert lib.grpo_async_advantage_from_stats(fake, fake, fake, 4, 2, 0.0, None, fake, fake, fake, fake,
                                               None) == L.GRPO_ERR_INVALID_ARG
