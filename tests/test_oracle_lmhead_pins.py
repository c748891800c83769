"""-m "not gpu": pins of the NEXT(2) oracle (oracle.run_batch_lmhead, logits = X W^T).

* one-hot hidden states make every logit an exact copy of a W entry, so the LM-head
  path must reproduce the logits path (already pinned) bit for bit;
* central finite differences of J with respect to X and W pin the chain rule
  (dJ/dX = dz W, dJ/dW = dz^T X -- a transposed or swapped operand fails).
"""
import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import f32_to_bf16_bits, make_manual

EPS32 = float(np.float32(0.2))


def _batch(rng, V, P=2, G=4, Lmax=4, K=3, lw=None, T=None):
    N = P * G
    L = rng.integers(1, Lmax + 1, size=N)
    g = rng.permutation(np.repeat(np.arange(P), G)).astype(np.int32)
    R = rng.integers(0, 3, size=N).astype(np.float32)
    ver = 1000 - rng.integers(1, K + 1, size=N)
    T = int(L.sum())
    tgt = rng.integers(0, V, size=T)
    return L, g, R, ver, T, tgt


@pytest.mark.parametrize("seed", range(4))
def test_onehot_hidden_reproduces_logits_path(seed):
    rng = np.random.default_rng(seed)
    V, d = 37, 16
    L, g, R, ver, T, tgt = _batch(rng, V)
    W = f32_to_bf16_bits((rng.normal(size=(V, d)) * 2).astype(np.float32))
    k = rng.integers(0, d, size=T)
    X = np.zeros((T, d), np.uint16)
    X[np.arange(T), k] = 0x3F80                                   # bf16 1.0
    z_bits = np.ascontiguousarray(W[:, k].T)                      # z[t, v] = W[v, k_t]
    lw = (rng.normal(size=T) * 0.5 - 3.5).astype(np.float32)
    b = make_manual(2, 4, 3, V, L, g, R, ver, tgt, lw)
    ld = b.ld
    bits = np.zeros((T, ld), np.uint16)
    bits[:, :V] = z_bits
    ref = O.run_batch(b, bits)
    lm = O.run_batch_lmhead(b, X, W)
    assert np.array_equal(lm["logits"], O._bf16_to_f64(z_bits))
    assert lm["J"] == ref["J"]
    for f in ("lse", "logp", "r", "term", "s"):
        assert np.array_equal(getattr(lm["rows"], f), getattr(ref["rows"], f)), f
    assert np.array_equal(lm["rows"].dlogits, ref["rows"].dlogits)


@pytest.mark.parametrize("seed", range(3))
def test_lmhead_gradients_finite_differences(seed):
    """-dJ/dX and -dJ/dW (Z19 sign) vs central differences, h = 1e-5."""
    rng = np.random.default_rng(50 + seed)
    V, d = int(rng.integers(3, 9)), int(rng.integers(2, 6))
    L, g, R, ver, T, tgt = _batch(rng, V)
    X = f32_to_bf16_bits(rng.normal(size=(T, d)).astype(np.float32))
    W = f32_to_bf16_bits(rng.normal(size=(V, d)).astype(np.float32))
    X64, W64 = O._bf16_to_f64(X), O._bf16_to_f64(W)
    z = X64 @ W64.T
    cur = (z - np.log(np.exp(z).sum(1, keepdims=True)))[np.arange(T), tgt]
    for _ in range(200):   # behaviour log-probs away from the clip kinks (J smooth around X, W)
        lw = (cur - rng.normal(size=T) * 0.25).astype(np.float32)
        r = np.exp(cur - lw.astype(np.float64))
        if np.all(np.abs(r - (1 + EPS32)) > 1e-3) and np.all(np.abs(r - (1 - EPS32)) > 1e-3):
            break
    b = make_manual(2, 4, 3, V, L, g, R, ver, tgt, lw)
    out = O.run_batch_lmhead(b, X, W)
    adv, inv = out["adv"], out["inv_norm"]

    def J(Xf, Wf):
        rr = O.rows_f64(np.arange(T), Xf @ Wf.T, tgt, lw, b.cu_seqlens, adv, inv, 0.2,
                        want_dlogits=False)
        return O.objective_tokens(b.cu_seqlens, inv, rr.term)[0]

    h = 1e-5
    for M, grad, which in ((X64, out["dhidden"], 0), (W64, out["dW"], 1)):
        num = np.zeros_like(M)
        for i in range(M.shape[0]):
            for j in range(M.shape[1]):
                Mp, Mm = M.copy(), M.copy()
                Mp[i, j] += h
                Mm[i, j] -= h
                Jp = J(Mp, W64) if which == 0 else J(X64, Mp)
                Jm = J(Mm, W64) if which == 0 else J(X64, Mm)
                num[i, j] = -(Jp - Jm) / (2 * h)
        err = np.abs(num - grad).max() / max(np.abs(grad).max(), 1e-12)
        assert err < 1e-6, (which, err)


def test_blockwise_helpers():
    """The block-wise full-size helpers are the same definitions: lmhead_logits_rows equals
    lmhead_logits bit for bit (each block holds the whole d-sum of its columns), and
    matmul_rows_W of one-hot rows returns rows of W exactly."""
    rng = np.random.default_rng(3)
    X = f32_to_bf16_bits(rng.normal(size=(5, 24)).astype(np.float32))
    W = f32_to_bf16_bits(rng.normal(size=(70, 24)).astype(np.float32))
    assert np.array_equal(O.lmhead_logits_rows(X, W, block=16), O.lmhead_logits(X, W))
    onehot = np.zeros((3, 70))
    onehot[0, 5] = onehot[1, 69] = onehot[2, 33] = 1.0
    got = O.matmul_rows_W(onehot, W, block=16)
    assert np.array_equal(got, O._bf16_to_f64(W)[[5, 69, 33]])
