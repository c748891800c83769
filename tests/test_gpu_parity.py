"""-m gpu: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs: bit-exact integers, logp within 2e-3 abs, loss within 1e-5
(guarded relative, Z17), dlogits within 1e-2 relative L2."""
import numpy as np
import pytest
import torch

from synth.gen import CONFIGS, f32_to_bf16_bits, make_batch, make_manual
from paper_2604_26256_b200._lib import GRPO_ERR_INVALID_ARG
from tests.gpu_util import compare, run_gpu, run_oracle, to_dev_bits

pytestmark = pytest.mark.gpu

# the row-wise kernel K3b, the ring kernel K3c with 16 KB slots, and the production
# instantiation of K3c (stream_kernel<512, 1, 2048, 1>, the auto plan for V >= 90000)
KERNELS = [{"kernel": 2}, {"kernel": 3}, {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3}]
KERNEL_IDS = ["rowwise", "stream16", "stream32"]
STREAM_PLANS = [{"kernel": 3, "stages": st, "lag": lg, "ctas_per_sm": nt, "chunk_kb": kb, "row_cache": cps}
                for st, lg, nt, kb, cps in ((13, 3, 0, 16, 0), (13, 1, 0, 16, 0), (13, 12, 0, 16, 0),
                                            (2, 1, 0, 16, 0), (5, 2, 0, 16, 0), (8, 3, 256, 16, 0),
                                            (13, 3, 256, 16, 0), (6, 3, 0, 32, 0), (6, 1, 0, 32, 0),
                                            (2, 1, 0, 32, 0), (6, 5, 0, 32, 0), (3, 1, 256, 32, 0),
                                            (7, 3, 0, 32, 0), (7, 2, 0, 32, 0), (7, 6, 0, 32, 0), (14, 3, 0, 16, 0),
                                            # two CTAs per SM (the auto plan for 34000 <= V < 90000)
                                            (6, 3, 256, 16, 2), (6, 1, 0, 16, 2), (3, 1, 0, 32, 2),
                                            (2, 1, 256, 32, 2))]
ROWWISE_PLANS = [{"kernel": 2, "ctas_per_sm": c, "stages": u, "row_cache": rc, "cluster_size": cl}
                 for c, u, rc, cl in ((1, 4, -1, 1), (1, 2, 0, 1), (1, 8, 1, 1), (2, 4, -1, 1),
                                      (2, 4, 0, 1), (2, 8, 1, 1), (2, 8, 0, 1), (2, 2, 0, 1),
                                      (3, 4, 2, 1), (3, 8, 0, 1), (4, 8, 0, 1), (8, 4, -1, 1),
                                      (8, 4, 0, 1), (2, 8, 0, 2), (1, 4, 0, 2), (4, 8, 0, 2),
                                      (2, 8, 0, 4), (2, 4, 3, 4))]


def _case(name, seed, **kw):
    b = make_batch(name, seed)
    bits = b.logits_bits()
    return b, bits


@pytest.mark.parametrize("tune", KERNELS, ids=KERNEL_IDS)
@pytest.mark.parametrize("seed", range(8))
def test_tiny_full_parity(dev, tune, seed):
    b, bits = _case("tiny", seed)
    ref = run_oracle(b, bits)
    gpu = run_gpu(b, bits, dev, tune=tune)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("tune", KERNELS, ids=KERNEL_IDS)
@pytest.mark.parametrize("name", ["mid32k", "mid152k", "ragged", "large_small"])
def test_config_parity(dev, tune, name):
    b, bits = _case(name, 1)
    ref = run_oracle(b, bits)
    gpu = run_gpu(b, bits, dev, tune=tune)
    errs = compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    print(name, tune, errs)


def test_retired_and_invalid_tunes_refused(dev):
    """Kernel 1 (the cluster-resident K3a) is retired, and tunes no kernel implements are
    host-side argument errors (GRPO_ERR_INVALID_ARG), not CUDA errors."""
    import paper_2604_26256_b200 as Gp
    b, bits = _case("ragged", 2)
    for tune in ({"kernel": 1}, {"kernel": 3, "cluster_size": 4}, {"kernel": 3, "cluster_size": 2,
                 "ctas_per_sm": 256}, {"kernel": 2, "cluster_size": 8}, {"kernel": 3, "stages": 40},
                 {"kernel": 3, "chunk_kb": 32, "stages": 8}):
        with pytest.raises(Gp.GrpoError) as ei:
            run_gpu(b, bits, dev, tune=tune)
        assert ei.value.status == GRPO_ERR_INVALID_ARG, (tune, ei.value)


@pytest.mark.parametrize("plan", ROWWISE_PLANS,
                         ids=lambda d: f"cps{d['ctas_per_sm']}u{d['stages']}c{d['row_cache']}"
                                       f"C{d['cluster_size']}")
def test_rowwise_plans(dev, plan):
    """Every row-wise kernel instantiation (threads x vectors in flight) matches the oracle."""
    for name in ("ragged", "mid152k"):
        b, bits = _case(name, 6)
        ref = run_oracle(b, bits)
        gpu = run_gpu(b, bits, dev, tune=plan)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    gpu = run_gpu(b, bits, dev, tune=dict(plan, prefetch=1))
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_chunked_equals_oracle(dev, chunks):
    """Trajectories straddling chunk boundaries keep their full-L weight."""
    b, bits = _case("mid32k", 3)
    ref = run_oracle(b, bits)
    gpu = run_gpu(b, bits, dev, chunks=chunks)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("tune", KERNELS, ids=KERNEL_IDS)
def test_inplace_and_forward_only(dev, tune):
    b, bits = _case("ragged", 4)
    ref = run_oracle(b, bits)
    gpu = run_gpu(b, bits, dev, tune=tune, inplace=True)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    fwd = run_gpu(b, bits, dev, tune=tune, want_dlogits=False)
    compare(fwd, ref, b, check_dlogits=False)
    assert np.array_equal(fwd["logp"], gpu["logp"])


def test_unfused_bwd_matches_fused(dev):
    """loss_bwd from the saved lse / token_scale reproduces the fused dlogits (<= 1 bf16 ulp)."""
    b, bits = _case("mid152k", 5)
    gpu = run_gpu(b, bits, dev)
    lg = to_dev_bits(bits, dev)
    out = torch.full_like(lg, 0x7FC3)
    import paper_2604_26256_b200 as G
    G.grpo_async_loss_bwd(lg, b.T, b.V, b.ld, torch.from_numpy(b.target_ids).to(dev),
                          torch.from_numpy(gpu["lse"].astype(np.float32)).to(dev),
                          torch.from_numpy(gpu["scale"].astype(np.float32)).to(dev), 1.0, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint16).astype(np.int32)
    fused = gpu["dlogits_raw"].astype(np.int32)
    # lse is handed over in natural units (the fused kernel keeps it in log2 units),
    # so the two may differ by one bf16 ulp on a few elements
    diff = np.abs(got - fused)
    assert diff.max() <= 1
    assert (diff != 0).mean() < 1e-3


def _adversarial_batch(V, rows):
    """One group of 4; rows given explicitly as float32 logits (rounded to bf16)."""
    T = len(rows)
    L = [T // 4] * 3 + [T - 3 * (T // 4)]
    tgt = np.array([r[1] for r in rows], np.int64)
    z = np.stack([r[0] for r in rows]).astype(np.float32)
    bits = f32_to_bf16_bits(z)
    zz = bits.astype(np.uint32) << 16
    zf = zz.view(np.float32).astype(np.float64)
    # behaviour log-probs: near-on-policy with a spread of ratios
    with np.errstate(over="ignore", invalid="ignore"):
        m = np.max(zf, 1, keepdims=True)
        lse = (m + np.log(np.sum(np.exp(zf - m), 1, keepdims=True)))[:, 0]
    cur = zf[np.arange(T), tgt] - lse
    rng = np.random.default_rng(0)
    lw = np.minimum(cur + rng.normal(size=T) * 0.2, 0).astype(np.float32)
    b = make_manual(1, 4, 1, V, L, [0, 0, 0, 0], [1, 0, 0.5, 0.25], [999] * 4, tgt, lw)
    pad = np.zeros((T, b.ld), np.uint16)
    pad[:, :V] = bits
    return b, pad


def test_adversarial_rows(dev):
    V = 4099  # V % 8 == 3
    rng = np.random.default_rng(1)
    rows = []
    rows.append((np.zeros(V), 0))                              # uniform row, target col 0
    rows.append((np.zeros(V), V - 1))                          # uniform, target in the ragged tail
    z = rng.normal(size=V); z[17] = 60.0; rows.append((z, 17))  # dominant entry (p ~ 1)
    z = rng.normal(size=V); z[17] = 60.0; rows.append((z, 5))   # dominant, other target
    z = rng.normal(size=V); z[::3] = -np.inf; rows.append((z, 1))  # masked vocabulary
    z = rng.normal(size=V) * 30; rows.append((z, 100))          # large magnitude
    z = rng.normal(size=V) + 1e4; rows.append((z, 7))           # large offset (bf16 coarse)
    z = np.full(V, -1e30); z[V - 2] = 0.0; rows.append((z, V - 2))  # one finite-dominant entry
    for _ in range(8):
        rows.append((rng.normal(size=V) * 3, int(rng.integers(0, V))))
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    for tune in KERNELS + [{"kernel": 2, "cluster_size": 4, "ctas_per_sm": 2}]:
        gpu = run_gpu(b, bits, dev, tune=tune)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("V", [40000, 152064])
def test_scale_jumps_along_the_row(dev, V):
    """Rows whose later chunks lie far above their first ones: the row-wise kernels keep
    the first finite batch's max as the exponent reference and raise it only when a
    thread's partial sum passes 2^64 (rowwise.cuh), so jumps below, at and above that
    threshold and above fp32's exp2 range (2^128) must all match the oracle."""
    rng = np.random.default_rng(11)
    rows = []
    for jump in (20.0, 40.0, 85.0, 200.0, 1e4):  # nats; 2^64 ~ e^44.4, 2^128 ~ e^88.7
        if jump < 1e4:  # (a target 1e4 below the max: logp = -1e4, Z23)
            z = rng.normal(size=V); z[V // 2:] += jump
            rows.append((z, int(rng.integers(0, V // 2))))  # target in the low half
        z = rng.normal(size=V); z[V // 2:] += jump
        rows.append((z, int(rng.integers(V // 2, V))))  # target in the high half
    z = np.linspace(-150.0, 150.0, V); rows.append((z, V - 3))  # steady climb
    z = np.full(V, -np.inf); z[-5:] = rng.normal(size=5); rows.append((z, V - 1))  # finite only at the end
    z = rng.normal(size=V) * 40; rows.append((z, 9))
    z = rng.normal(size=V); z[-1] = 120.0; rows.append((z, 0))  # one late dominant entry
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    for tune in KERNELS:
        gpu = run_gpu(b, bits, dev, tune=tune)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])


def test_single_token_trajectories_and_empty_chunk(dev):
    rng = np.random.default_rng(3)
    V, P, G = 300, 2, 4
    L = np.ones(P * G, np.int64)
    T = int(L.sum())
    g = np.repeat(np.arange(P), G)
    tgt = rng.integers(0, V, T)
    lw = -rng.uniform(3, 8, T).astype(np.float32)
    b = make_manual(P, G, 1, V, L, g, rng.integers(0, 2, P * G), [999] * (P * G), tgt, lw)
    bits = np.zeros((T, b.ld), np.uint16)
    bits[:, :V] = f32_to_bf16_bits(rng.normal(size=(T, V)).astype(np.float32))
    ref = run_oracle(b, bits)
    for chunks in (1, T + 3):  # includes empty chunks
        gpu = run_gpu(b, bits, dev, chunks=chunks)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])


def test_validate_faults_bitexact(dev):
    """Injected faults (T5) through the C ABI against the oracle, bit for bit."""
    import oracle.oracle as O
    base = make_batch("stale_small" if "stale_small" in CONFIGS else "ragged", 0)
    cases = []
    for gap in (base.K, base.K + 1, -1, 0):
        v = base.version_ids.copy(); v[1] = base.v_theta - gap
        cases.append(dict(version_ids=v))
    g = base.group_ids.copy(); g[0] = base.P; cases.append(dict(group_ids=g))
    g = base.group_ids.copy(); g[0] = -3; cases.append(dict(group_ids=g))
    t = base.target_ids.copy(); t[5] = base.V; t[9] = -1; cases.append(dict(target_ids=t))
    lw = base.logp_behav.copy(); lw[3] = 0.25; lw[11] = np.nan; lw[12] = -np.inf
    cases.append(dict(logp_behav=lw))
    cu = base.cu_seqlens.copy(); cu[2] = cu[1]; cases.append(dict(cu_seqlens=cu))
    cases.append(dict(tbs=base.tbs + 1))
    tv = np.repeat(base.version_ids, base.lengths); tv[0] -= 1
    cases.append(dict(token_version=tv))
    for case in cases:
        b = make_batch("ragged", 0)
        for k, val in case.items():
            setattr(b, k, val)
        bits = np.zeros((b.T, b.ld), np.uint16)
        ref = O.validate(b.version_ids, b.cu_seqlens, b.group_ids, b.target_ids, P=b.P, V=b.V,
                         G=b.G, tbs=b.tbs, v_theta=b.v_theta, K=b.K,
                         token_version=b.token_version, logp_behav=b.logp_behav)
        import paper_2604_26256_b200 as Gp
        db = Gp.DeviceBatch.from_host(b, dev)
        vo = Gp.GrpoAsyncLoss().validate(db)
        torch.cuda.synchronize()
        assert np.array_equal(vo.traj_flags.cpu().numpy().view(np.uint32), ref["traj_flags"]), case
        assert np.array_equal(vo.group_count.cpu().numpy(), ref["group_count"]), case
        assert np.array_equal(vo.stale_hist.cpu().numpy().reshape(b.P, b.K + 1), ref["stale_hist"])
        assert vo.summary_dict() == ref["summary"], case
        assert ref["summary"]["valid"] == 0 or case.get("version_ids") is not None


@pytest.mark.parametrize("R", [2, 4, 8])
def test_sharded_equals_unsharded(dev, R):
    """T6: LPT shards processed one after another on one GPU (rank-local packing,
    replicated advantages through traj_index) reproduce the unsharded result:
    integer counters exact, J within fp64 reordering, per-row values bit-identical."""
    import paper_2604_26256_b200 as Gp
    b, bits = _case("mid32k", 7)
    full = run_gpu(b, bits, dev)
    db = Gp.DeviceBatch.from_host(b, dev)
    loss = Gp.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    stats = torch.zeros(Gp.NUM_STATS, dtype=torch.float64, device=dev)
    logp = np.full(b.T, np.nan)
    traj_sum = np.zeros(b.N)
    for mine in Gp.lpt_partition(b.lengths, R):
        rows, cu_l = Gp.shard_rows(b.cu_seqlens, mine)
        lg = to_dev_bits(bits[rows], dev)
        ts = torch.zeros(len(mine), dtype=torch.float64, device=dev)
        lp = torch.empty(len(rows), device=dev)
        loss.loss_chunk(lg, 0, len(rows), torch.from_numpy(b.target_ids[rows]).to(dev),
                        torch.from_numpy(b.logp_behav[rows]).to(dev),
                        torch.from_numpy(cu_l).to(dev), adv, inv, ts, stats,
                        traj_index=torch.from_numpy(mine.astype(np.int32)).to(dev),
                        logp_out=lp, V=b.V)
        torch.cuda.synchronize()
        logp[rows] = lp.cpu().numpy()
        traj_sum[mine] = ts.cpu().numpy()
    st = stats.cpu().numpy()
    for k in (Gp.STAT_ROWS, Gp.STAT_CLIPPED, Gp.STAT_ACTIVE):
        assert st[k] == full["stats"][k]
    assert abs(st[Gp.STAT_J] - full["stats"][Gp.STAT_J]) <= 1e-12 * full["stats"][Gp.STAT_ABS]
    assert np.array_equal(logp.astype(np.float32), full["logp"].astype(np.float32))
    assert np.array_equal(traj_sum, full["traj_sum"])


@pytest.mark.parametrize("plan", STREAM_PLANS,
                         ids=lambda d: f"ns{d['stages']}pf{d['lag']}nt{d['ctas_per_sm'] or 512}"
                                       f"kb{d['chunk_kb']}cps{d['row_cache'] or 1}"
                                       f"kb{d['chunk_kb']}")
def test_stream_plans(dev, plan):
    """K3c (one row per SM through the bulk-copy ring) for ring sizes from 2 slots (every
    chunk but one re-loaded) to 13 (rows shorter than the ring: several rows resident),
    out-of-place and forward-only, against the oracle."""
    for name in ("tiny", "ragged", "mid152k"):
        b, bits = _case(name, 8)
        ref = run_oracle(b, bits)
        gpu = run_gpu(b, bits, dev, tune=plan, chunks=2)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    ref = run_oracle(b, bits, want_dlogits=False)
    gpu = run_gpu(b, bits, dev, tune=plan, want_dlogits=False)
    compare(gpu, ref, b, check_dlogits=False)


@pytest.mark.parametrize("V", [2, 7, 8, 9, 100, 16391, 32776, 34003, 50689, 90007])
def test_odd_vocabulary_sizes(dev, V):
    """Small and ragged vocabularies (V % 8 != 0; one vector past a 16 KB / 32 KB ring slot;
    the K3b/K3c switch point) for the row-wise and both ring geometries."""
    rng = np.random.default_rng(V)
    rows = [(rng.normal(size=V) * 2, int(rng.integers(0, V))) for _ in range(12)]
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    for tune in ({"kernel": 2}, {"kernel": 3}, {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3},
                 {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 1}, None):
        gpu = run_gpu(b, bits, dev, tune=tune)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])


def test_auto_plan_choice(dev):
    """The auto plan (tune kernel 0): K3b below V = 34000, K3c with two 256-thread CTAs per
    SM and 16 KB slots up to V = 90000, K3c with one CTA per SM and 32 KB slots from there
    on (7 slots, one free at the end of pass 1), each
    row split over a two-CTA cluster (the same ring) from
    V = 240000 (DESIGN.md section 8 measurements); an explicitly tuned call is never
    redirected."""
    import paper_2604_26256_b200 as Gp
    for V, kernel, cps in ((30000, 2, None), (34000, 3, 2), (76032, 3, 2), (89990, 3, 2),
                           (90000, 3, 1), (152064, 3, 1), (163840, 3, 1), (163848, 3, 1), (239999, 3, 1),
                           (240000, 3, 1), (262144, 3, 1)):
        rows = [(np.random.default_rng(V).normal(size=V), 3) for _ in range(4)]
        b, bits = _adversarial_batch(V, rows)
        ref = run_oracle(b, bits)
        gpu = run_gpu(b, bits, dev)
        plan = Gp.grpo_async_last_plan()
        assert plan["kernel"] == kernel, (V, plan)
        if kernel == 3:
            ns = 6 if cps == 2 else 7
            assert plan["stages"] == ns and plan["ctas_per_sm"] == cps, (V, plan)
            assert plan["smem_bytes"] >= ns * (32768 if cps == 1 else 16384)
            assert plan["vec_per_thread"] == (512 if cps == 1 else 256), (V, plan)
            assert plan["cluster_size"] == (2 if V >= 240000 else 1), (V, plan)
            if cps == 1:
                assert plan["lag"] == 1, (V, plan)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    run_gpu(b, bits, dev, tune={"kernel": 2, "stages": 8})
    assert Gp.grpo_async_last_plan()["kernel"] == 2


@pytest.mark.parametrize("name", ["mid152k", "large_small"])
def test_inplace_auto_plan_long_rows(dev, name):
    """In-place dlogits (dlogits == logits) with the auto plan on long rows (K3c, 32 KB slots:
    pass 2 writes the resident chunks while the re-loads of the row's head are in flight)."""
    b, bits = _case(name, 4)
    ref = run_oracle(b, bits)
    gpu = run_gpu(b, bits, dev, inplace=True, chunks=2)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("name", ["mid152k", "ragged", "large_small"])
def test_run_to_run_bitwise_determinism(dev, name):
    """Every reduction has a fixed order (per-thread partials, fixed block/warp trees, fp64
    segment sums in row order): two runs give identical bits for every output."""
    b, bits = _case(name, 11)
    g1 = run_gpu(b, bits, dev, chunks=3)
    g2 = run_gpu(b, bits, dev, chunks=3)
    for k in ("adv", "inv_norm", "logp", "lse", "scale", "traj_sum", "stats", "dlogits_raw"):
        assert np.array_equal(g1[k], g2[k], equal_nan=True), k


def test_step_captures_into_a_cuda_graph(dev):
    """One step of the path (validate, advantage, fused loss over row chunks) is stream-ordered
    with no host synchronisation, so it captures into a CUDA graph; replays reproduce the
    eager outputs bit for bit."""
    import paper_2604_26256_b200 as Gp
    b, bits = _case("mid152k", 12)
    eager = run_gpu(b, bits, dev, chunks=2)
    db = Gp.DeviceBatch.from_host(b, dev)
    loss = Gp.GrpoAsyncLoss()
    T, ld, V = b.T, b.ld, b.V
    lg = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(dev)
    dl = torch.full((T, ld), 0x7FC3, dtype=torch.int16, device=dev)
    logp = torch.empty(T, device=dev)
    traj_sum = torch.zeros(b.N, dtype=torch.float64, device=dev)
    stats = torch.zeros(Gp.NUM_STATS, dtype=torch.float64, device=dev)
    vo = Gp.ValidateOut(b.N, b.P, b.K, dev)
    adv = torch.empty(b.N, device=dev)
    inv = torch.empty(b.N, device=dev)
    loss.workspace(T - T // 2, V, b.N, dev)  # allocate outside the capture

    def step():
        traj_sum.zero_()
        stats.zero_()
        loss.validate(db, vo)
        loss.advantage(db, adv, inv)
        for r0, r1 in ((0, T // 2), (T // 2, T)):
            loss.loss_chunk(lg[r0:r1], r0, r1 - r0, db.target_ids[r0:r1], db.logp_behav[r0:r1],
                            db.cu_seqlens, adv, inv, traj_sum, stats, dlogits=dl[r0:r1],
                            logp_out=logp[r0:r1], V=V)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm-up on the side stream (function attributes, tensor maps)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(logp.cpu().numpy().astype(np.float64), eager["logp"])
    assert np.array_equal(stats.cpu().numpy(), eager["stats"])
    assert np.array_equal(traj_sum.cpu().numpy(), eager["traj_sum"])
    assert np.array_equal(dl.cpu().numpy().view(np.uint16), eager["dlogits_raw"])


@pytest.mark.parametrize("seed", range(10))
def test_random_shapes_and_plans(dev, seed):
    """Fuzz: random vocabulary size, row count, row padding and launch plan (row-wise,
    streamed ring with random slot size / count / free slots) against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.choice([int(rng.integers(2, 600)), int(rng.integers(600, 40000)),
                        int(rng.integers(40000, 200000))]))
    n = int(rng.integers(4, 48))
    rows = [(rng.normal(size=V) * float(rng.uniform(0.5, 4)), int(rng.integers(0, V))) for _ in range(n)]
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    kb = int(rng.choice([16, 24, 32, 48]))
    ns = int(rng.integers(2, 208 // kb + 1))
    plans = [None, {"kernel": 2}, {"kernel": 3, "chunk_kb": kb, "stages": ns,
                                   "lag": int(rng.integers(1, ns))}]
    for tune in plans:
        gpu = run_gpu(b, bits, dev, tune=tune, chunks=int(rng.integers(1, 4)),
                      inplace=bool(rng.integers(0, 2)))
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("seed", [188, 24, 73])
def test_precision_regression_cases(dev, seed):
    """The fuzz cases that bounded the loss precision (profiles/r02_precision_fuzz.txt): seed
    188 broke round 1's 1e-2 * S_abs guard (|J| = 1.2e-3 S_abs, 21 rows); 24 and 73 are the
    worst of 200 seeds for round 2 and round 1.  Every plan, the standard criteria (Z17)."""
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.choice([int(rng.integers(2, 600)), int(rng.integers(600, 40000)),
                        int(rng.integers(40000, 200000))]))
    n = int(rng.integers(4, 48))
    rows = [(rng.normal(size=V) * float(rng.uniform(0.5, 4)), int(rng.integers(0, V))) for _ in range(n)]
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    plans = [None, {"kernel": 2}, {"kernel": 3}, {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3}]
    if V >= 16384:
        plans.append({"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3, "cluster_size": 2})
    for tune in plans:
        gpu = run_gpu(b, bits, dev, tune=tune)
        errs = compare(gpu, ref, b, logits_pad=bits[:, b.V:])
        assert errs["J_rel_guarded"] <= 5e-6, (tune, errs["J_rel_guarded"])  # 2x inside the bound


SPLIT_PLANS = [{"kernel": 3, "cluster_size": 2, "chunk_kb": kb, "stages": ns, "lag": pf}
               for kb, ns, pf in ((32, 7, 1), (32, 7, 3), (32, 6, 3), (32, 6, 1), (32, 2, 1), (16, 13, 3),
                                  (16, 3, 2))]


@pytest.mark.parametrize("plan", SPLIT_PLANS,
                         ids=lambda d: f"kb{d['chunk_kb']}ns{d['stages']}pf{d['lag']}")
def test_stream_split_rows(dev, plan):
    """K3c with each row shared by a cluster of two CTAs (cluster_size 2, the DSMEM exchange
    of the two (max, sum) partials): configs with V = 152064 and 262144 in two chunks, forward
    only, and odd vocabularies whose halves end in a ragged vector, against the oracle."""
    for name in ("mid152k", "large_small"):
        b, bits = _case(name, 9)
        ref = run_oracle(b, bits)
        gpu = run_gpu(b, bits, dev, tune=plan, chunks=2)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    ref = run_oracle(b, bits, want_dlogits=False)
    gpu = run_gpu(b, bits, dev, tune=plan, want_dlogits=False)
    compare(gpu, ref, b, check_dlogits=False)
    for V in (16384, 16391, 32777, 90007):
        rng = np.random.default_rng(V)
        # targets in the first half, the second half, at both ends and on the split column
        h = (((V + 7) // 8 + 1) // 2) * 8
        tg = [0, V - 1, h - 1, h, int(rng.integers(0, V)), int(rng.integers(0, V)), h + 1, 5]
        rows = [(rng.normal(size=V) * 2, t) for t in tg]
        b, bits = _adversarial_batch(V, rows)
        ref = run_oracle(b, bits)
        gpu = run_gpu(b, bits, dev, tune=plan)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:])


def _dead_rows_batch(V, seed):
    """Four groups of four trajectories, interleaved in completion order: groups 0 and 2 have
    equal rewards (A = 0: dead rows), groups 1 and 3 mixed ones; lengths 1..6 tokens."""
    rng = np.random.default_rng(seed)
    P, G = 4, 4
    order = rng.permutation(P * G)
    group_ids = (order // G).astype(np.int32)
    rewards = np.where(group_ids == 0, 1.0, np.where(group_ids == 2, 0.0,
                                                     rng.integers(0, 2, P * G).astype(float)))
    for p in (1, 3):  # make sure the live groups are not all-equal
        i = np.nonzero(group_ids == p)[0]
        rewards[i[0]], rewards[i[1]] = 1.0, 0.0
    L = rng.integers(1, 7, P * G)
    T = int(L.sum())
    z = rng.normal(size=(T, V)).astype(np.float32) * 2.0
    tgt = rng.integers(0, V, T)
    bits = f32_to_bf16_bits(z)
    zf = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    m = zf.max(1, keepdims=True)
    lse = (m + np.log(np.exp(zf - m).sum(1, keepdims=True)))[:, 0]
    lw = np.minimum(zf[np.arange(T), tgt] - lse + rng.normal(size=T) * 0.2, 0).astype(np.float32)
    b = make_manual(P, G, 1, V, L, group_ids, rewards, [999] * (P * G), tgt, lw)
    pad = np.zeros((T, b.ld), np.uint16)
    pad[:, :V] = bits
    return b, pad


DEAD_PLANS = [None, {"kernel": 3}, {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3},
              {"kernel": 3, "chunk_kb": 32, "stages": 7, "lag": 3},
              {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 1},
              {"kernel": 3, "chunk_kb": 16, "stages": 13, "lag": 3},
              {"kernel": 3, "chunk_kb": 32, "stages": 2, "lag": 1},
              {"kernel": 3, "cluster_size": 2, "chunk_kb": 32, "stages": 6, "lag": 1},
              {"kernel": 3, "cluster_size": 2, "chunk_kb": 16, "stages": 3, "lag": 2}]


@pytest.mark.parametrize("V", [90007, 152064, 262144])
def test_stream_dead_rows(dev, V):
    """Runs of dead rows (A = 0, or a trajectory masked out: inv_norm = 0) between live
    ones through K3c's two-pass ring (re-loads at V >= 90007, split rows at 262144): a dead
    row's dlogits are zeros (its math-free pass 2), a live row's unaffected.  Element-wise
    against the oracle: every plan, row chunks 1 and 3, in place and not, the dlogits
    buffer pre-filled with NaN so a missing zero store would show."""
    b, bits = _dead_rows_batch(V, V)
    mask = np.ones(b.N, np.uint8)
    mask[np.nonzero(b.group_ids == 1)[0][0]] = 0  # one masked trajectory in a live group
    for traj_mask in (None, mask):
        ref = run_oracle(b, bits, traj_mask=traj_mask)
        assert np.any(ref["rows"].s == 0) and np.any(ref["rows"].s != 0)
        for k, tune in enumerate(DEAD_PLANS):
            gpu = run_gpu(b, bits, dev, tune=tune, chunks=1 + 2 * (k % 2), inplace=k % 3 == 1,
                          traj_mask=traj_mask)
            compare(gpu, ref, b, logits_pad=bits[:, b.V:])
