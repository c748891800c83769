"""synth/gen.py -- seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no log-softmax, no ratio,
no clipping, no advantage, no reduction of the objective).  It only draws
inputs with the shapes of the paper's workloads:

* lengths: uniform, or lognormal with a truncation spike at L_max
  (long-tailed CoT responses, PAPER.md P:52-66 fig:resp_in_house / _2,
  mean response 2.4K tokens P:284);
* prompt groups of G responses, rewards Bernoulli(q_p);
* behaviour versions: exactly K distinct staleness gaps, the longest
  trajectories the stalest (long tails outlive steps);
* optional per-token versions for partial-rollout style trajectories;
* bf16 logits from a counter-based generator (one element = one SplitMix64
  draw), shaped by a Zipf-like per-vocabulary base row;
* targets drawn from the Zipf base distribution, behaviour log-probs from
  the sampling distribution plus Gaussian drift that grows with staleness.

The same counter-based logits generator is implemented a second time in CUDA
(synth/csrc/synth_fill.cu) for device-side filling of large batches; the two
must agree bit for bit (tests/test_gpu_synth.py).  Every random number is a
pure function of (seed, stream, index).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)

# stream ids
S_LEN, S_LEN2, S_SPIKE, S_REWARD_Q, S_REWARD, S_LOGITS, S_TARGET, S_DELTA, S_DELTA2, \
    S_OUTLIER, S_PERM, S_PARTIAL, S_GAP = range(13)

V_THETA = 1000


def mix64(z):
    """SplitMix64 finaliser on uint64 numpy arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        z = (np.array([seed], np.uint64) * GOLDEN + np.array([stream], np.uint64) * STREAM_MUL
             + np.uint64(1))
    return mix64(z)[0]


def draw(key, idx):
    """uint64 draw number idx of the stream with this key."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(np.uint64(key) + (idx + np.uint64(1)) * GOLDEN)


def uniform(key, idx):
    """double in [0, 1) with 53 random bits."""
    return (draw(key, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed, stream_a, stream_b, idx):
    """Box-Muller standard normal (host only; never mirrored on the device)."""
    u1 = uniform(stream_key(seed, stream_a), idx)
    u2 = uniform(stream_key(seed, stream_b), idx)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * math.pi * u2)


# ----------------------------------------------------------------- logits
def f32_to_bf16_bits(x):
    """Round-to-nearest-even float32 -> bf16 bit pattern (finite inputs)."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (r & np.uint64(0xFFFF)).astype(np.uint16)


def bf16_bits_to_f32(bits):
    return (np.asarray(bits, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def logit_noise(key, phys_rows, V, cols=None):
    """float32 noise numerator c = (u0+u1+u2+u3) - 131070 for elements (row, col).

    One SplitMix64 draw per element at counter row*V + col; its four 16-bit
    lanes are summed as integers (Irwin-Hall(4), exact), then converted to
    float32 exactly.  Returned shape [len(rows), len(cols)].
    """
    rows = np.asarray(phys_rows, np.uint64).reshape(-1, 1)
    c = np.arange(V, dtype=np.uint64) if cols is None else np.asarray(cols, np.uint64)
    c = c.reshape(1, -1) if cols is None else c.reshape(rows.shape[0], -1)
    with np.errstate(over="ignore"):
        h = draw(key, rows * np.uint64(V) + c)
    m = np.uint64(0xFFFF)
    s = (h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48))
    return (s.astype(np.int64) - 131070).astype(np.float32)


@dataclass
class LogitsSpec:
    """Counter-based bf16 logits:  z[t, v] = bf16_rn(base[v] + scale * c(t mod period, v)).

    Both products/sums are single IEEE float32 operations (no FMA), which the
    CUDA twin reproduces with __fmul_rn / __fadd_rn.
    """
    key: np.uint64
    base: np.ndarray          # float32 [V]
    scale: np.float32         # sigma * sqrt(3) / 65536
    period: int               # logical row t reads physical row t % period

    def rows_bits(self, rows, cols=None):
        rows = np.asarray(rows, np.int64)
        phys = (rows % self.period).astype(np.uint64)
        c = logit_noise(self.key, phys, len(self.base), cols)
        a = (c * self.scale).astype(np.float32)               # RN multiply
        if cols is None:
            z = (self.base[None, :] + a).astype(np.float32)    # RN add
        else:
            z = (self.base[np.asarray(cols, np.int64)].reshape(a.shape) + a).astype(np.float32)
        return f32_to_bf16_bits(z)

    def noise_at(self, rows, cols):
        """The float32 a = scale*c at (row, col) pairs (used for behaviour log-probs)."""
        rows = np.asarray(rows, np.int64)
        phys = (rows % self.period).astype(np.uint64)
        c = logit_noise(self.key, phys, len(self.base), np.asarray(cols).reshape(-1, 1))
        return (c.reshape(-1) * self.scale).astype(np.float32)


# ----------------------------------------------------------------- configs
@dataclass
class Config:
    name: str
    P: int
    G: int
    K: int
    V: int
    length: tuple               # ("uniform", lo, hi) | ("lognormal", mean, sigma, lmax, p_spike)
    logits: str = "zipf"        # "iid" | "zipf"
    sigma_logit: float = 0.15   # per-element logit noise std
    zipf_alpha: float = 1.5
    sigma0: float = 0.03        # behaviour drift std per unit of (1 + gap)
    outlier_p: float = 1e-3
    partial_frac: float = 0.0   # fraction of above-median trajectories with per-token versions
    g0: int = 1                 # smallest staleness gap (1 = one-step off-policy pipeline)
    ld_pad: int = 0             # extra padding columns (ld = round_up(V, 8) + ld_pad)
    eps: float = 0.2
    std_floor: float = 1e-8
    note: str = ""


CONFIGS = {
    # BASELINE.json configs[0..4]
    "tiny": Config("tiny", 1, 8, 2, 1024, ("uniform", 4, 64), logits="iid", sigma_logit=2.0,
                   sigma0=0.15, note="BJ configs[0]"),
    "dapo": Config("dapo", 32, 16, 2, 152064, ("lognormal", 2400.0, 1.0, 20000, 0.0),
                   note="BJ configs[1] DAPO-Math-17K-shaped"),
    "stale": Config("stale", 64, 8, 8, 152064, ("lognormal", 2000.0, 1.0, 20000, 0.0),
                    partial_frac=0.25, note="BJ configs[2] high staleness + partial rollout"),
    "prod": Config("prod", 128, 16, 3, 152064, ("lognormal", 330.0, 1.3, 32768, 0.005),
                   note="BJ configs[3] production long tail, ~1M tokens"),
    "large": Config("large", 256, 8, 4, 262144, ("lognormal", 1000.0, 1.2, 65536, 0.002),
                    note="BJ configs[4] large-vocab stress"),
    # parity-test shapes (oracle finishes in seconds; several tiles + ragged tails)
    "mid32k": Config("mid32k", 4, 8, 3, 32000, ("lognormal", 60.0, 1.0, 400, 0.02),
                     sigma0=0.1, note="V=32k, several clusters per row"),
    "mid152k": Config("mid152k", 2, 4, 2, 152064, ("lognormal", 40.0, 1.0, 200, 0.05),
                      sigma0=0.1, note="the metric's vocab at oracle-friendly T"),
    "ragged": Config("ragged", 3, 4, 4, 50257, ("lognormal", 30.0, 1.0, 120, 0.05),
                     sigma0=0.1, ld_pad=24, partial_frac=0.5,
                     note="V % 8 != 0, padded ld, mixed token versions"),
    "large_small": Config("large_small", 2, 4, 4, 262144, ("lognormal", 20.0, 1.0, 80, 0.0),
                          sigma0=0.1, note="V=256k at oracle-friendly T"),
}


@dataclass
class Batch:
    cfg: Config
    seed: int
    P: int
    G: int
    K: int
    V: int
    ld: int
    tbs: int
    v_theta: int
    cu_seqlens: np.ndarray      # int64 [N+1]
    group_ids: np.ndarray       # int32 [N]
    version_ids: np.ndarray     # int64 [N]
    token_version: np.ndarray | None  # int64 [T] or None
    rewards: np.ndarray         # float32 [N]
    target_ids: np.ndarray      # int64 [T]
    logp_behav: np.ndarray      # float32 [T]
    lengths: np.ndarray         # int64 [N]
    logits: LogitsSpec = field(repr=False, default=None)

    @property
    def N(self):
        return len(self.group_ids)

    @property
    def T(self):
        return int(self.cu_seqlens[-1])

    def logits_bits(self, rows=None):
        rows = np.arange(self.T) if rows is None else rows
        out = np.zeros((len(rows), self.ld), np.uint16)
        for b in range(0, len(rows), 256):
            out[b:b + 256, :self.V] = self.logits.rows_bits(rows[b:b + 256])
        return out


def _lengths(cfg: Config, seed: int, N: int) -> tuple[np.ndarray, np.ndarray]:
    idx = np.arange(N)
    kind = cfg.length[0]
    spike = np.zeros(N, bool)
    if kind == "uniform":
        lo, hi = cfg.length[1], cfg.length[2]
        L = lo + (draw(stream_key(seed, S_LEN), idx) % np.uint64(hi - lo + 1)).astype(np.int64)
    elif kind == "lognormal":
        mean, sigma, lmax, p_spike = cfg.length[1:]
        mu = math.log(mean) - sigma * sigma / 2.0
        z = normal(seed, S_LEN, S_LEN2, idx)
        L = np.clip(np.rint(np.exp(mu + sigma * z)), 1, lmax).astype(np.int64)
        spike = uniform(stream_key(seed, S_SPIKE), idx) < p_spike
        L[spike] = lmax
    else:
        raise ValueError(kind)
    return L, spike


def zipf_base(cfg: Config, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """base[v] = -alpha * ln(1 + rank(v)), rank a seeded permutation; also rank->vocab map."""
    V = cfg.V
    keys = draw(stream_key(seed, S_PERM), np.arange(V))
    order = np.argsort(keys, kind="stable")           # order[rank] = vocab id
    rank = np.empty(V, np.int64)
    rank[order] = np.arange(V)
    base = (-cfg.zipf_alpha * np.log1p(rank.astype(np.float64))).astype(np.float32)
    return base, order


def make_batch(cfg: Config | str, seed: int = 0, period: int | None = None) -> Batch:
    """Draw one synthetic training batch (metadata on the host; logits lazily by spec)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    P, G, K, V = cfg.P, cfg.G, cfg.K, cfg.V
    N = P * G
    L0, spike0 = _lengths(cfg, seed, N)
    group0 = np.arange(N) // G
    # rewards: q_p ~ U(0,1) per prompt, R_i ~ Bernoulli(q_p); truncated responses get 0
    q = uniform(stream_key(seed, S_REWARD_Q), np.arange(P))
    R0 = (uniform(stream_key(seed, S_REWARD), np.arange(N)) < q[group0]).astype(np.float32)
    R0[spike0] = 0.0
    # staleness gaps: exactly K distinct values, longest trajectories stalest
    rank = np.empty(N, np.int64)
    rank[np.lexsort((np.arange(N), L0))] = np.arange(N)
    qi = rank / N
    gap0 = cfg.g0 + np.minimum(K - 1, np.floor(K * qi).astype(np.int64))
    # completion order: stalest first, then shorter first, then index
    order = np.lexsort((np.arange(N), L0, -gap0))
    L, group_ids, R, gap = L0[order], group0[order].astype(np.int32), R0[order], gap0[order]
    version_ids = (V_THETA - gap).astype(np.int64)
    cu = np.zeros(N + 1, np.int64)
    cu[1:] = np.cumsum(L)
    T = int(cu[-1])
    tok_traj = np.repeat(np.arange(N), L)
    tok_gap = gap[tok_traj].copy()
    token_version = None
    if cfg.partial_frac > 0:
        token_version = version_ids[tok_traj].copy()
        med = np.median(L)
        pick = uniform(stream_key(seed, S_PARTIAL), np.arange(N)) < cfg.partial_frac
        for i in np.nonzero(pick & (L > med) & (L >= 3))[0]:
            h = draw(stream_key(seed, S_PARTIAL), np.array([N + 3 * i, N + 3 * i + 1, N + 3 * i + 2]))
            nseg = 2 + int(h[0] % np.uint64(2))
            cuts = sorted(set(int(1 + x % np.uint64(L[i] - 1)) for x in h[1:nseg]))
            b = cu[i]
            bounds = [0] + cuts + [int(L[i])]
            for s in range(len(bounds) - 1):
                v = min(int(version_ids[i]) + s, V_THETA)
                token_version[b + bounds[s]:b + bounds[s + 1]] = v
        tok_gap = V_THETA - token_version
    # logits spec
    lkey = stream_key(seed, S_LOGITS)
    if cfg.logits == "iid":
        base = np.zeros(V, np.float32)
        vocab_of_rank = None
        log_norm = math.log(V)
    else:
        base, vocab_of_rank = zipf_base(cfg, seed)
        log_norm = math.log(np.sum(np.exp(base.astype(np.float64))))  # Zipf normaliser sum_j (1+j)^-alpha
    scale = np.float32(cfg.sigma_logit * math.sqrt(3.0) / 65536.0)
    spec = LogitsSpec(lkey, base, scale, period if period else max(T, 1))
    # targets: uniform (iid) or from the Zipf sampling distribution by inverse CDF
    u = uniform(stream_key(seed, S_TARGET), np.arange(T))
    if vocab_of_rank is None:
        target_ids = np.minimum((u * V).astype(np.int64), V - 1)
    else:
        w = np.exp(-cfg.zipf_alpha * np.log1p(np.arange(V, dtype=np.float64)))
        cdf = np.cumsum(w)
        j = np.minimum(np.searchsorted(cdf, u * cdf[-1], side="right"), V - 1)
        target_ids = vocab_of_rank[j].astype(np.int64)
    # behaviour log-probs: log q(y) + the generator's own noise at y, minus a
    # constant normaliser estimate (log_norm + sigma^2/2), minus a staleness drift
    a_y = spec.noise_at(np.arange(T), target_ids).astype(np.float64) if T else np.zeros(0)
    drift = normal(seed, S_DELTA, S_DELTA2, np.arange(T)) * cfg.sigma0 * (1.0 + tok_gap)
    uo = uniform(stream_key(seed, S_OUTLIER), np.arange(2 * T))
    out = uo[:T] < cfg.outlier_p
    drift[out] = np.where(uo[T:][out] < 0.5, -1.0, 1.0) * (1.0 + 4.0 * uo[:T][out] / cfg.outlier_p)
    lw = base[target_ids].astype(np.float64) + a_y - log_norm - cfg.sigma_logit ** 2 / 2.0 - drift
    logp_behav = np.minimum(lw, 0.0).astype(np.float32)
    ld = ((V + 7) // 8) * 8 + cfg.ld_pad
    return Batch(cfg, seed, P, G, K, V, ld, N, V_THETA, cu, group_ids, version_ids,
                 token_version, R.astype(np.float32), target_ids, logp_behav, L, spec)


def make_manual(P, G, K, V, lengths, group_ids, rewards, version_ids, target_ids, logp_behav,
                token_version=None, v_theta=V_THETA, tbs=None, ld=None) -> Batch:
    """Wrap hand-written arrays (adversarial / hand-worked cases) as a Batch (no logits spec)."""
    L = np.asarray(lengths, np.int64)
    cu = np.zeros(len(L) + 1, np.int64)
    cu[1:] = np.cumsum(L)
    return Batch(None, -1, P, G, K, V, ld or ((V + 7) // 8) * 8, len(L) if tbs is None else tbs,
                 v_theta, cu, np.asarray(group_ids, np.int32), np.asarray(version_ids, np.int64),
                 None if token_version is None else np.asarray(token_version, np.int64),
                 np.asarray(rewards, np.float32), np.asarray(target_ids, np.int64),
                 np.asarray(logp_behav, np.float32), L, None)


def lmhead_inputs(T, V, d, seed, w_scale=2.5):
    """NEXT(2) inputs (TEST/BENCH INPUT GENERATOR): bf16 bit patterns of hidden states
    X [T, d] ~ N(0, 1) and an LM-head weight W [V, d] ~ N(0, (w_scale / sqrt(d))^2), so the
    logits z = X W^T have a standard deviation of about w_scale (DESIGN.md input recipe)."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 0x4C4D]))
    X = f32_to_bf16_bits(rng.standard_normal((T, d), dtype=np.float32))
    W = f32_to_bf16_bits(rng.standard_normal((V, d), dtype=np.float32) *
                         np.float32(w_scale / np.sqrt(d)))
    return X, W
