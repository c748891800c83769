"""Host-side checks of the seeded input generator (synth/gen.py), -m "not gpu"."""
import math

import numpy as np
import pytest

from synth.gen import CONFIGS, f32_to_bf16_bits, make_batch, stream_key, draw


def test_bf16_rounding_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(size=100000).astype(np.float32) * 10,
                        np.array([0.0, -0.0, 1e-40, 3.0e38, 1.00390625, 1.01171875], np.float32)])
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(f32_to_bf16_bits(x), ref)


def test_splitmix_reference_values():
    """SplitMix64 (Steele et al.): state 0 -> first output 0xE220A8397B1DCDAF."""
    from synth.gen import mix64, GOLDEN
    assert int(mix64(np.array([GOLDEN], np.uint64))[0]) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("name", list(CONFIGS))
def test_batch_shapes_and_determinism(name):
    cfg = CONFIGS[name]
    b1 = make_batch(name, 0)
    b2 = make_batch(name, 0)
    assert b1.N == cfg.P * cfg.G and b1.tbs == b1.N
    assert np.array_equal(b1.cu_seqlens, b2.cu_seqlens)
    assert np.array_equal(b1.logp_behav, b2.logp_behav)
    assert np.all(np.bincount(b1.group_ids, minlength=cfg.P) == cfg.G)
    gaps = b1.v_theta - b1.version_ids
    assert sorted(set(gaps.tolist())) == list(range(cfg.g0, cfg.g0 + cfg.K))
    assert b1.target_ids.min() >= 0 and b1.target_ids.max() < cfg.V
    assert np.all(b1.logp_behav <= 0) and np.all(np.isfinite(b1.logp_behav))
    assert b1.ld % 8 == 0 and b1.ld >= cfg.V
    if cfg.length[0] == "lognormal":
        assert b1.lengths.max() <= cfg.length[3]


def test_lognormal_length_law():
    """Monte Carlo vs closed form: mean of the untruncated lognormal body."""
    from synth.gen import Config, _lengths
    cfg = Config("x", 1, 1, 1, 8, ("lognormal", 2400.0, 1.0, 10 ** 9, 0.0))
    L, _ = _lengths(cfg, 0, 200000)
    assert abs(L.mean() / 2400.0 - 1) < 0.02
    mu = math.log(2400.0) - 0.5
    assert abs(np.median(L) / math.exp(mu) - 1) < 0.02


def test_logits_rows_repeat_with_period():
    b = make_batch("mid32k", 0, period=100)
    a = b.logits.rows_bits([5, 105, 205])
    assert np.array_equal(a[0], a[1]) and np.array_equal(a[0], a[2])
