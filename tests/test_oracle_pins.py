"""Pins of the fp64 oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the oracle function(s) it pins and what pins it: a worked
example (tests/golden/*.json, cited), a closed form, an invariant, a library
routine on a special case, brute force or finite differences.  None of them
re-types the oracle's formula.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import f32_to_bf16_bits, make_batch, make_manual

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EPS32 = float(np.float32(0.2))


def _golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- O2 advantage
def test_advantage_spec_examples():
    """O2 vs SPEC worked examples S:528-530 (golden/spec_examples.json)."""
    for ex in _golden("spec_examples.json")["group_advantage"]:
        R = ex["rewards"]
        adv, inv, gc = O.advantage(R, [0] * len(R), np.arange(len(R) + 1), 1)
        assert gc[0] == len(R)
        np.testing.assert_allclose(adv, ex["expected"], rtol=0, atol=ex["tol"] + 1e-300)
        if ex["tol"] == 0.0:
            assert np.all(adv == 0.0)


def test_advantage_exact_sqrt_three_halves():
    """[2,0,1]: mean 1, population std sqrt(2/3) -> A = +-sqrt(3/2) (closed form, Z1)."""
    adv, _, _ = O.advantage([2, 0, 1], [0, 0, 0], [0, 1, 2, 3], 1)
    assert abs(adv[0] - math.sqrt(1.5)) < 1e-15 and abs(adv[1] + math.sqrt(1.5)) < 1e-15
    assert adv[2] == 0.0


def test_advantage_degenerate_group_is_exactly_zero():
    """Z2: bitwise-equal rewards give A = 0 exactly even when the fp64 mean is inexact."""
    adv, _, _ = O.advantage([0.1, 0.1, 0.1], [0, 0, 0], [0, 1, 2, 3], 1)
    assert np.all(adv == 0.0)
    adv, _, gc = O.advantage([0.5], [0], [0, 4], 1)      # single member
    assert adv[0] == 0.0 and gc[0] == 1


@pytest.mark.parametrize("seed", range(20))
def test_advantage_invariants(seed):
    """Sum A = 0 per group, population std of A = 1, shift/scale invariance."""
    rng = np.random.default_rng(seed)
    P, G = 5, int(rng.integers(2, 17))
    N = P * G
    g = rng.permutation(np.repeat(np.arange(P), G)).astype(np.int32)
    R = rng.normal(size=N).astype(np.float32)
    cu = np.concatenate([[0], np.cumsum(rng.integers(1, 9, size=N))])
    adv, inv, gc = O.advantage(R, g, cu, P)
    assert np.all(gc == G)
    for p in range(P):
        a = adv[g == p]
        assert abs(a.sum()) < 1e-12
        assert abs(np.sqrt(np.mean(a * a)) - 1.0) < 1e-12
    # shift by an exactly representable constant
    adv2, _, _ = O.advantage(R + np.float32(3.0), g, cu, P)
    np.testing.assert_allclose(adv2, adv, atol=1e-6)   # R+3 rounds in float32
    Ri = rng.integers(0, 8, size=N).astype(np.float32)  # integer rewards: shift/scale exact
    a1, _, _ = O.advantage(Ri, g, cu, P)
    a2, _, _ = O.advantage(Ri + 5, g, cu, P)
    a3, _, _ = O.advantage(Ri * 4, g, cu, P)
    np.testing.assert_allclose(a2, a1, atol=1e-12)
    np.testing.assert_allclose(a3, a1, atol=1e-12)


def test_advantage_unbiased_closed_form():
    """NEXT(1) sample std: [2,0,1] has sample std 1 -> A = (+1, -1, 0) exactly; a binary
    group of G with k ones has A_i = (R_i - k/G) / sqrt(k(G-k)/(G(G-1)))."""
    adv, _, _ = O.advantage([2, 0, 1], [0, 0, 0], [0, 1, 2, 3], 1, unbiased=True)
    assert list(adv) == [1.0, -1.0, 0.0]
    G, k = 8, 3
    R = np.array([1.0] * k + [0.0] * (G - k), np.float32)
    adv, _, _ = O.advantage(R, [0] * G, np.arange(G + 1), 1, unbiased=True)
    sd = math.sqrt(k * (G - k) / (G * (G - 1)))
    np.testing.assert_allclose(adv[:k], (1 - k / G) / sd, rtol=1e-14)
    np.testing.assert_allclose(adv[k:], (0 - k / G) / sd, rtol=1e-14)


@pytest.mark.parametrize("seed", range(5))
def test_advantage_unbiased_vs_numpy_ddof1(seed):
    """Against numpy's sample std (ddof=1) per group; the single-member group and the
    bitwise-equal group keep A = 0; unbiased = population * sqrt((n-1)/n)."""
    rng = np.random.default_rng(100 + seed)
    P, G = 6, int(rng.integers(2, 12))
    g = rng.permutation(np.repeat(np.arange(P), G)).astype(np.int32)
    R = rng.normal(size=P * G).astype(np.float32)
    g = np.concatenate([g, [P]]).astype(np.int32)          # group P: one member
    R = np.concatenate([R, np.float32([0.7])])
    R[g == 0] = np.float32(0.25)                           # group 0: bitwise equal
    cu = np.arange(len(R) + 1)
    a_u, _, gc = O.advantage(R, g, cu, P + 1, unbiased=True)
    a_p, _, _ = O.advantage(R, g, cu, P + 1)
    assert gc[P] == 1 and a_u[g == P][0] == 0.0 and np.all(a_u[g == 0] == 0.0)
    for p in range(1, P):
        m = g == p
        r = R[m].astype(np.float64)
        np.testing.assert_allclose(a_u[m], (r - r.mean()) / np.std(r, ddof=1), rtol=1e-12,
                                   atol=1e-14)
        np.testing.assert_allclose(a_u[m], a_p[m] * math.sqrt((G - 1) / G), rtol=1e-12,
                                   atol=1e-14)


def test_inv_norm_weights_sum_to_one():
    """inv_norm_i = 1/(P G_p L_i): sum_i inv_norm_i * L_i = 1 (each prompt weighs 1/P, Z5)."""
    b = make_batch("mid32k", 3)
    _, inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P)
    assert abs(np.sum(inv * b.lengths) - 1.0) < 1e-12


# ----------------------------------------------------------------- O4 token
def test_clipped_term_spec_examples():
    """O4 vs SPEC S:535-537.  eps arrives as float32 and is widened (1+eps = 1.2000000030)."""
    for ex in _golden("spec_examples.json")["clipped_term"]:
        r, term, clipped, s = O.token(math.log(ex["r"]), 0.0, ex["A"], 1.0, ex["eps"])
        assert abs(r - ex["r"]) < 1e-15
        assert abs(term - ex["expected"]) < 1e-8


def test_token_branches_and_gradient_flow():
    """O4 case analysis: clipped iff the clip branch is strictly smaller; ties flow (Z10)."""
    hi, lo = 1.0 + EPS32, 1.0 - EPS32
    cases = [  # (r, A, clipped, expected term)
        (1.5, 1.0, True, hi), (1.5, -1.0, False, -1.5), (0.5, 1.0, False, 0.5),
        (0.5, -1.0, True, -lo), (1.0, 2.0, False, 2.0), (1.1, -3.0, False, -3.3),
        (2.0, 0.0, False, 0.0)]
    for r, A, clipped, exp_term in cases:
        rr, term, c, s = O.token(math.log(r), 0.0, A, 0.5, 0.2)
        assert c == clipped, (r, A)
        assert abs(term - exp_term) < 1e-12
        assert s == (0.0 if clipped else 0.5 * A * rr)
    # exact tie at the boundary: the clip value equals r, gradient flows
    _, term, c, s = O.token(math.log(hi), 0.0, 1.0, 1.0, 0.2)
    assert abs(term - hi) < 1e-12


# ----------------------------------------------------------------- O3 log-softmax
def test_log_softmax_vs_torch():
    """O3 vs torch.log_softmax in fp64 on random bf16 rows (library routine)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    for V in (1, 2, 7, 100, 1024, 5000):
        z = (rng.normal(size=V) * 3).astype(np.float32)
        bits = f32_to_bf16_bits(z)
        zz = torch.from_numpy(bits.astype(np.int32) << 16).view(torch.float32).double()
        ref = torch.log_softmax(zz, dim=0)
        for y in {0, V - 1, V // 2}:
            lse, logp = O.log_softmax_row(bits, y)
            assert abs(logp - ref[y].item()) < 1e-12
            assert abs(lse - torch.logsumexp(zz, 0).item()) < 1e-12


def test_log_softmax_closed_forms():
    """HW6: uniform row -> logp = -ln V.  HW7: z_y = M, others 0 -> p_y = e^M/(e^M+V-1)."""
    for V in (4, 1000, 152064):
        for c in (0.0, 5.0, -30.0):
            bits = f32_to_bf16_bits(np.full(V, c, np.float32))
            lse, logp = O.log_softmax_row(bits, V // 3)
            assert abs(logp + math.log(V)) < 1e-12 * max(1, math.log(V))
            assert abs(lse - (c + math.log(V))) < 1e-11
    for V, M in ((10, 3.0), (152064, 12.0), (1024, -4.0)):
        z = np.zeros(V, np.float32)
        z[7] = M
        lse, logp = O.log_softmax_row(f32_to_bf16_bits(z), 7)
        # sequential fp64 sum over V terms: rounding grows like V * 2^-53
        assert abs(logp - (M - math.log(math.exp(M) + V - 1))) < 1e-13 + 1e-16 * V


def test_log_softmax_shift_invariance_and_masking():
    """Integer rows + integer c (exact in bf16) leave logp unchanged; -inf entries have p = 0."""
    rng = np.random.default_rng(1)
    z = rng.integers(-64, 65, size=3000).astype(np.float32)
    for c in (-17.0, 3.0, 64.0):
        _, a = O.log_softmax_row(f32_to_bf16_bits(z), 11)
        _, b = O.log_softmax_row(f32_to_bf16_bits(z + c), 11)
        assert abs(a - b) < 1e-12
    zm = np.full(64, -np.inf, np.float32)
    zm[:4] = 0.0
    _, logp = O.log_softmax_row(f32_to_bf16_bits(zm), 2)
    assert abs(logp + math.log(4)) < 1e-15


# ----------------------------------------------------------------- O5 gradient
def test_dlogits_row_invariants():
    """O5: rows sum to 0, the target entry has sign -s, others sign s; s = 0 gives exact zeros."""
    rng = np.random.default_rng(2)
    bits = f32_to_bf16_bits((rng.normal(size=2000) * 2).astype(np.float32))
    lse, _ = O.log_softmax_row(bits, 5)
    for s in (0.37, -1.3e-5):
        d = O.dlogits_row(bits, 5, lse, s)
        assert abs(d.sum()) < 1e-12 * abs(s) * 10
        assert np.sign(d[5]) == -np.sign(s)
        assert np.all(np.sign(np.delete(d, 5)) == np.sign(s))
    assert np.all(O.dlogits_row(bits, 5, lse, 0.0) == 0.0)


def _tiny_batch(rng, P=2, G=4, V=6, Lmax=4, K=3):
    N = P * G
    L = rng.integers(1, Lmax + 1, size=N)
    g = rng.permutation(np.repeat(np.arange(P), G)).astype(np.int32)
    R = rng.integers(0, 3, size=N).astype(np.float32)
    ver = 1000 - rng.integers(1, K + 1, size=N)
    T = int(L.sum())
    tgt = rng.integers(0, V, size=T)
    return L, g, R, ver, T, tgt


def _J_of(z, b, adv, inv, eps=0.2):
    rr = O.rows_f64(np.arange(b.T), z, b.target_ids, b.logp_behav, b.cu_seqlens, adv, inv, eps,
                    want_dlogits=False)
    J, _ = O.objective_tokens(b.cu_seqlens, inv, rr.term)
    return J


@pytest.mark.parametrize("seed", range(6))
def test_gradient_finite_differences(seed):
    """O5 (and O3/O4 through it) vs central finite differences of J (h = 1e-5), V <= 16.

    Tokens within 1e-3 of a clip kink are re-drawn so J is smooth around z.
    dlogits is d(-J)/dz (Z19).
    """
    rng = np.random.default_rng(100 + seed)
    V = int(rng.integers(2, 17))
    L, g, R, ver, T, tgt = _tiny_batch(rng, V=V)
    z = rng.normal(size=(T, V)) * 1.5
    # behaviour log-probs near the current ones, away from the clip kinks
    lsm = z - np.log(np.exp(z).sum(1, keepdims=True))
    cur = lsm[np.arange(T), tgt]
    for _ in range(100):
        lw = (cur - rng.normal(size=T) * 0.25).astype(np.float32)
        r = np.exp(cur - lw.astype(np.float64))
        if np.all(np.abs(r - (1 + EPS32)) > 1e-3) and np.all(np.abs(r - (1 - EPS32)) > 1e-3):
            break
    b = make_manual(2, 4, 3, V, L, g, R, ver, tgt, lw)
    adv, inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P)
    rr = O.rows_f64(np.arange(T), z, tgt, lw, b.cu_seqlens, adv, inv, 0.2)
    h = 1e-5
    num = np.zeros_like(z)
    for t in range(T):
        for v in range(V):
            zp = z.copy(); zp[t, v] += h
            zm = z.copy(); zm[t, v] -= h
            num[t, v] = -(_J_of(zp, b, adv, inv) - _J_of(zm, b, adv, inv)) / (2 * h)
    err = np.abs(num - rr.dlogits).max() / max(np.abs(rr.dlogits).max(), 1e-12)
    assert err < 1e-6, err
    # with noise 0.25 on the ratios, every seed clips some tokens (zero-gradient rows, whose
    # finite differences are zero too) and keeps others active
    assert rr.clipped.any() and (~rr.clipped).any()


def test_gradient_vs_torch_autograd():
    """O5 vs torch fp64 autograd of the PPO-clip surrogate built from torch primitives
    (log_softmax, gather, clamp, minimum) on a random batch away from clip kinks."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    V = 12
    L, g, R, ver, T, tgt = _tiny_batch(rng, V=V, Lmax=6)
    z = rng.normal(size=(T, V)) * 2
    lsm = z - np.log(np.exp(z).sum(1, keepdims=True))
    cur = lsm[np.arange(T), tgt]
    lw = (cur - rng.normal(size=T) * 0.3).astype(np.float32)
    r = np.exp(cur - lw.astype(np.float64))
    keep = (np.abs(r - (1 + EPS32)) > 1e-6) & (np.abs(r - (1 - EPS32)) > 1e-6)
    assert keep.all()
    b = make_manual(2, 4, 3, V, L, g, R, ver, tgt, lw)
    adv, inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P)
    rr = O.rows_f64(np.arange(T), z, tgt, lw, b.cu_seqlens, adv, inv, 0.2)
    zt = torch.tensor(z, dtype=torch.float64, requires_grad=True)
    traj = torch.tensor(np.repeat(np.arange(len(L)), L))
    A = torch.tensor(adv)[traj]
    w = torch.tensor(inv)[traj]
    logp = torch.log_softmax(zt, 1).gather(1, torch.tensor(tgt).view(-1, 1)).squeeze(1)
    rt = torch.exp(logp - torch.tensor(lw, dtype=torch.float64))
    surr = torch.minimum(rt * A, torch.clamp(rt, 1 - EPS32, 1 + EPS32) * A)
    J = (w * surr).sum()
    (-J).backward()
    np.testing.assert_allclose(rr.dlogits, zt.grad.numpy(), atol=1e-13, rtol=1e-10)
    J_or, _ = O.objective_tokens(b.cu_seqlens, inv, rr.term)
    assert abs(J_or - J.item()) < 1e-13


# ----------------------------------------------------------------- O4 objective
def _hw3_batch():
    hw = _golden("hw3.json")
    V = hw["V"]
    ratios = [x for traj in hw["ratios"] for x in traj]
    T = len(ratios)
    lw = np.array([-math.log(4) - math.log(x) for x in ratios], np.float32)
    b = make_manual(1, 4, 1, V, hw["lengths"], [0, 0, 0, 0], hw["rewards"], [1000] * 4,
                    [1] * T, lw, v_theta=1000)
    z = np.zeros((T, V), np.uint16)      # bf16 bits of 0.0
    return hw, b, z


def test_hw3_hand_worked_batch():
    """HW3 (golden/hw3.json): the full path on a hand-worked batch."""
    hw, b, z = _hw3_batch()
    e = hw["expected"]
    res = O.run_batch(b, z, eps=hw["eps"])
    tol = hw["tol"]
    np.testing.assert_allclose(res["adv"], e["adv"], atol=1e-15)
    M = res["traj_sum"] / b.lengths
    np.testing.assert_allclose(M, e["M"], atol=tol)
    assert abs(res["J"] - e["J"]) < tol
    assert list(res["rows"].clipped) == e["clipped"]
    np.testing.assert_allclose(res["rows"].s, e["s"], atol=tol)
    dl = res["rows"].dlogits
    for k in range(b.T):
        d = e["dlogits_nonzero_rows"].get(str(k))
        if d is None:
            assert np.all(dl[k] == 0.0)
        else:
            assert abs(dl[k, 1] - d["target_value"]) < tol
            np.testing.assert_allclose(np.delete(dl[k], 1), d["non_target"], atol=tol)
    assert res["validate"]["summary"]["valid"] == 1


def test_hw4_constant_ratio_closed_form():
    """HW4: constant r on every token.  J = 0 inside the trust region, and outside
    J = (1/P) sum_p S_p+ (1+eps-r)/G_p  (r > 1+eps), (1/P) sum_p S_p+ (r-1+eps)/G_p (r < 1-eps),
    with S_p+ the sum of positive advantages.  R = [1,0,0,1], r = 1.5 or 0.5 -> J = -0.15."""
    for r_const, expect in ((1.5, -0.15), (0.5, -0.15), (1.1, 0.0), (0.9, 0.0)):
        V, L = 8, [3, 1, 2, 5]
        T = sum(L)
        lw = np.full(T, -math.log(V) - math.log(r_const), np.float32)
        b = make_manual(1, 4, 1, V, L, [0] * 4, [1, 0, 0, 1], [1000] * 4, [3] * T, lw)
        res = O.run_batch(b, np.zeros((T, V), np.uint16), eps=0.2, want_dlogits=False)
        assert abs(res["J"] - expect) < 1e-6, (r_const, res["J"])


def test_hw5_on_policy_and_sync_special_case():
    """HW5: logp_w = logp_theta gives r = 1 (exactly, uniform rows) and J = 0 because advantages
    are zero-mean per group; a single-version batch (K = 1) is the sync objective eq:grpo."""
    for seed in range(5):
        rng = np.random.default_rng(seed)
        P, G, V = 3, 4, 16
        L = rng.integers(1, 9, size=P * G)
        T = int(L.sum())
        lw = np.full(T, -math.log(V), np.float32)
        g = rng.permutation(np.repeat(np.arange(P), G))
        b = make_manual(P, G, 1, V, L, g, rng.integers(0, 2, P * G), [999] * (P * G),
                        rng.integers(0, V, T), lw)
        res = O.run_batch(b, np.zeros((T, V), np.uint16))
        r = res["rows"].r
        assert np.all(np.abs(r - 1.0) < 1e-7)
        S_abs = np.sum(res["inv_norm"][np.repeat(np.arange(P * G), L)] * np.abs(res["rows"].term))
        assert abs(res["J"]) <= 1e-7 * S_abs


@pytest.mark.parametrize("name,seed", [("tiny", s) for s in range(5)] + [("ragged", 0), ("mid32k", 1)])
def test_nested_triple_loop_equals_token_form(name, seed):
    """O4: the per-token weighted sum equals the literal nested sum over prompts ->
    versions B_j -> trajectories -> tokens of eq:grpo_async to 1e-12."""
    b = make_batch(name, seed)
    rng = np.random.default_rng(seed)
    term = rng.normal(size=b.T)
    _, inv, _ = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P)
    J1, _ = O.objective_tokens(b.cu_seqlens, inv, term)
    J2 = O.objective_nested(b.cu_seqlens, b.group_ids, b.version_ids, term, b.P)
    assert abs(J1 - J2) < 1e-12 * max(1.0, abs(J1))


# ----------------------------------------------------------------- O1 validate
def _clean_batch():
    return make_batch("tiny", 0)


def _val(b, **kw):
    args = dict(P=b.P, V=b.V, G=b.G, tbs=b.tbs, v_theta=b.v_theta, K=b.K,
                token_version=b.token_version, logp_behav=b.logp_behav)
    args.update(kw)
    return O.validate(b.version_ids, b.cu_seqlens, b.group_ids, b.target_ids, **args)


def test_validate_clean_batch_and_histogram():
    """O1 on a generated batch: valid, counts = G, |B_j| histogram sums to G (sum_j |B_j| = G, P:7)."""
    for name in ("tiny", "mid32k", "mid152k"):
        b = make_batch(name, 0)
        v = _val(b)
        assert v["rc"] == 0 and v["summary"]["valid"] == 1
        assert np.all(v["group_count"] == b.G)
        assert np.all(v["stale_hist"].sum(1) == b.G)
        assert v["summary"]["max_staleness"] == b.K and v["summary"]["min_staleness"] == 1
        assert np.all(v["traj_flags"] == 0)


def test_validate_injected_faults():
    """O1 vs injected faults (brute force by construction): each fault sets exactly its bit on
    exactly the faulted trajectory; gap = K passes (inclusive bound, Z8)."""
    b = _clean_batch()
    K = b.K
    # gap = K passes, K + 1 fails (STALE), gap < 0 fails (FUTURE)
    for gap, bit in ((K, 0), (K + 1, 1 << 0), (-1, 1 << 1), (0, 0)):
        ver = b.version_ids.copy()
        ver[3] = b.v_theta - gap
        v = O.validate(ver, b.cu_seqlens, b.group_ids, b.target_ids, P=b.P, V=b.V, G=b.G,
                       tbs=b.tbs, v_theta=b.v_theta, K=K)
        exp = np.zeros(b.N, np.uint32)
        exp[3] = bit
        assert np.array_equal(v["traj_flags"], exp), gap
        assert v["summary"]["c3_ok"] == (bit == 0)
    # bad group id -> BAD_GROUP_ID on that traj, GROUP_SIZE on the rest of its group (G-1 members)
    g = b.group_ids.copy()
    g[2] = b.P
    v = O.validate(b.version_ids, b.cu_seqlens, g, b.target_ids, P=b.P, V=b.V, G=b.G, tbs=b.tbs,
                   v_theta=b.v_theta, K=K)
    assert v["traj_flags"][2] == (1 << 3)
    assert np.all(np.delete(v["traj_flags"], 2) == (1 << 4))
    assert v["summary"]["c2_dropped"] == 1 and v["summary"]["c2_ok"] == 0
    # target out of range, logp_behav > 0 and NaN
    tg = b.target_ids.copy()
    tg[b.cu_seqlens[5] + 1] = b.V
    lw = b.logp_behav.copy()
    lw[b.cu_seqlens[6]] = 0.5
    lw[b.cu_seqlens[1]] = np.nan
    v = O.validate(b.version_ids, b.cu_seqlens, b.group_ids, tg, P=b.P, V=b.V, G=b.G, tbs=b.tbs,
                   v_theta=b.v_theta, K=K, logp_behav=lw)
    exp = np.zeros(b.N, np.uint32)
    exp[5] = 1 << 6
    exp[6] = 1 << 7
    exp[1] = 1 << 7
    assert np.array_equal(v["traj_flags"], exp)
    # mixed token versions (C1)
    tv = np.repeat(b.version_ids, b.lengths)
    tv[b.cu_seqlens[4]] += 1
    v = O.validate(b.version_ids, b.cu_seqlens, b.group_ids, b.target_ids, P=b.P, V=b.V, G=b.G,
                   tbs=b.tbs, v_theta=b.v_theta, K=K, token_version=tv)
    exp = np.zeros(b.N, np.uint32)
    exp[4] = 1 << 5
    assert np.array_equal(v["traj_flags"], exp)
    assert v["summary"]["n_c1_mixed"] == 1
    # zero-length trajectory, TBS mismatch
    cu = b.cu_seqlens.copy()
    cu[3] = cu[2]
    v = O.validate(b.version_ids, cu, b.group_ids, b.target_ids, P=b.P, V=b.V, G=b.G,
                   tbs=b.tbs + 8, v_theta=b.v_theta, K=K)
    assert v["traj_flags"][2] == (1 << 2)
    assert v["summary"]["tbs_ok"] == 0 and v["summary"]["valid"] == 0


def test_validate_group_size_brute_force():
    """G-1 and G+1 members: every member of the off-size group carries GROUP_SIZE."""
    rng = np.random.default_rng(5)
    for delta in (-1, +1):
        P, G = 3, 4
        g = np.repeat(np.arange(P), G)
        if delta < 0:
            g = g[1:]
        else:
            g = np.concatenate([[0], g])
        N = len(g)
        L = rng.integers(1, 5, size=N)
        cu = np.concatenate([[0], np.cumsum(L)])
        v = O.validate(np.full(N, 999), cu, g, np.zeros(cu[-1], np.int64), P=P, V=4, G=G,
                       tbs=P * G, v_theta=1000, K=1)
        for i in range(N):
            assert bool(v["traj_flags"][i] & (1 << 4)) == (g[i] == 0)
        assert v["summary"]["n_groups_wrong_size"] == 1
        assert v["summary"]["c2_dropped"] == (1 if delta < 0 else 0)


# ----------------------------------------------------------------- NEXT(1): DAPO options
def _const_ratio_batch(r_const, V=8, L=(3, 1, 2, 5)):
    T = sum(L)
    lw = np.full(T, -math.log(V) - math.log(r_const), np.float32)
    return make_manual(1, 4, 1, V, L, [0] * 4, [1, 0, 0, 1], [1000] * 4, [3] * T, lw), T, V


def test_clip_higher_closed_form():
    """Asymmetric clip [1-eps_lo, 1+eps_hi] (DAPO clip-higher): constant ratio r on every
    token of R = [1,0,0,1] gives per-trajectory means min(rA, clip(r)A) in closed form:
      r = 1.5:  A>0 -> 1+eps_hi, A<0 -> -r          J = (2(1+eps_hi) - 2r)/4
      r = 1.25, eps_hi = 0.28: inside the range -> J = 0 (symmetric eps = 0.2 gives -0.025)
      r = 0.5:  A>0 -> r, A<0 -> -(1-eps_lo)         J = (2r - 2(1-eps_lo))/4"""
    hi = float(np.float32(0.28))
    lo = float(np.float32(0.2))
    for r_const, eps_hi, expect in ((1.5, 0.28, (2 * (1 + hi) - 3.0) / 4), (1.25, 0.28, 0.0),
                                    (1.25, 0.2, (2 * (1 + lo) - 2.5) / 4),
                                    (0.5, 0.28, (1.0 - 2 * (1 - lo)) / 4)):
        b, T, V = _const_ratio_batch(r_const)
        res = O.run_batch(b, np.zeros((T, V), np.uint16), eps=0.2, eps_hi=eps_hi, want_dlogits=False)
        assert abs(res["J"] - expect) < 1e-6, (r_const, eps_hi, res["J"], expect)


def test_token_mean_weights():
    """Token-mean normalisation (DAPO): w_i = 1/sum of kept L; with equal lengths it coincides with
    the paper's sequence mean 1/(P G L); kept weights always satisfy sum_i w_i L_i = 1."""
    rng = np.random.default_rng(11)
    P, G = 3, 4
    g = rng.permutation(np.repeat(np.arange(P), G)).astype(np.int32)
    cu = np.arange(P * G + 1) * 7
    _, inv, gc = O.advantage(np.zeros(P * G, np.float32), g, cu, P)
    w_tok = O.weights(g, cu, gc, P, norm=1)
    np.testing.assert_allclose(w_tok, inv, rtol=1e-15)
    np.testing.assert_allclose(w_tok, 1.0 / cu[-1], rtol=1e-15)
    L = rng.integers(1, 20, size=P * G)
    cu = np.concatenate([[0], np.cumsum(L)])
    mask = (rng.random(P * G) < 0.7).astype(np.uint8)
    _, _, gc = O.advantage(np.zeros(P * G, np.float32), g, cu, P)
    w = O.weights(g, cu, gc, P, norm=1, traj_mask=mask)
    assert abs(np.sum(w * L) - 1.0) < 1e-12
    assert np.all(w[mask == 0] == 0.0)
    ws = O.weights(g, cu, gc, P, norm=0, traj_mask=mask)
    _, inv, _ = O.advantage(np.zeros(P * G, np.float32), g, cu, P)
    np.testing.assert_allclose(ws, np.where(mask == 1, inv, 0.0), rtol=1e-15)


def test_mask_equals_sub_batch():
    """Masking every trajectory outside one prompt group equals running that group as its own
    batch (groups are independent, eq:group_advantage; token mean over the kept tokens)."""
    b = make_batch("mid32k", 4)
    bits = b.logits_bits()
    p0 = 2
    mask = (b.group_ids == p0).astype(np.uint8)
    full = O.run_batch(b, bits, norm=1, traj_mask=mask, want_dlogits=False)
    idx = np.nonzero(mask)[0]
    rows = np.concatenate([np.arange(b.cu_seqlens[i], b.cu_seqlens[i + 1]) for i in idx])
    sub = make_manual(1, b.G, b.K, b.V, b.lengths[idx], np.zeros(len(idx), np.int32),
                      b.rewards[idx], b.version_ids[idx], b.target_ids[rows], b.logp_behav[rows])
    ref = O.run_batch(sub, bits[rows], norm=1, want_dlogits=False)
    assert abs(full["J"] - ref["J"]) < 1e-12 * max(1.0, abs(ref["J"]))


@pytest.mark.parametrize("seed", range(3))
def test_gradient_finite_differences_dapo(seed):
    """O5 under clip-higher + token-mean weights + a trajectory mask vs central differences;
    masked trajectories get exactly zero gradient."""
    rng = np.random.default_rng(300 + seed)
    V = int(rng.integers(2, 12))
    L, g, R, ver, T, tgt = _tiny_batch(rng, V=V)
    z = rng.normal(size=(T, V)) * 1.5
    lsm = z - np.log(np.exp(z).sum(1, keepdims=True))
    cur = lsm[np.arange(T), tgt]
    hi = float(np.float32(0.28))
    for _ in range(100):
        lw = (cur - rng.normal(size=T) * 0.25).astype(np.float32)
        r = np.exp(cur - lw.astype(np.float64))
        if np.all(np.abs(r - (1 + hi)) > 1e-3) and np.all(np.abs(r - (1 - EPS32)) > 1e-3):
            break
    b = make_manual(2, 4, 3, V, L, g, R, ver, tgt, lw)
    adv, _, gc = O.advantage(b.rewards, b.group_ids, b.cu_seqlens, b.P)
    mask = np.ones(len(L), np.uint8)
    mask[int(rng.integers(0, len(L)))] = 0
    w = O.weights(b.group_ids, b.cu_seqlens, gc, b.P, norm=1, traj_mask=mask)
    rr = O.rows_f64(np.arange(T), z, tgt, lw, b.cu_seqlens, adv, w, 0.2, eps_hi=0.28)

    def J_of(zz):
        q = O.rows_f64(np.arange(T), zz, tgt, lw, b.cu_seqlens, adv, w, 0.2, eps_hi=0.28,
                       want_dlogits=False)
        return O.objective_tokens(b.cu_seqlens, w, q.term)[0]
    h = 1e-5
    num = np.zeros_like(z)
    for t in range(T):
        for v in range(V):
            zp = z.copy(); zp[t, v] += h
            zm = z.copy(); zm[t, v] -= h
            num[t, v] = -(J_of(zp) - J_of(zm)) / (2 * h)
    err = np.abs(num - rr.dlogits).max() / max(np.abs(rr.dlogits).max(), 1e-12)
    assert err < 1e-6, err
    masked_rows = np.repeat(mask == 0, L)
    assert np.all(rr.dlogits[masked_rows] == 0.0)
