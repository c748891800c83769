"""-m gpu: NEXT(1) -- the DAPO loss options the paper trains with through
grpo_async_advantage_ex / grpo_async_loss_fwd_ex against the oracle: clip-higher
(eps_hi = 0.28), token-mean normalisation, and trajectory masks (overlong
responses, C1-violating partial rollouts)."""
import numpy as np
import pytest

import oracle.oracle as O
from synth.gen import make_batch
from tests.gpu_util import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

OPTS = [dict(eps_hi=0.28), dict(norm="token"), dict(eps_hi=0.28, norm="token")]


def _c1_mask(b):
    v = O.validate(b.version_ids, b.cu_seqlens, b.group_ids, b.target_ids, P=b.P, V=b.V, G=b.G,
                   tbs=b.tbs, v_theta=b.v_theta, K=b.K, token_version=b.token_version)
    return ((v["traj_flags"] & (1 << 5)) == 0).astype(np.uint8)


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("opts", OPTS, ids=["cliphigher", "tokenmean", "both"])
@pytest.mark.parametrize("name", ["mid32k", "mid152k"])
def test_dapo_options(dev, kernel, opts, name):
    b = make_batch(name, 2)
    bits = b.logits_bits()
    ref = run_oracle(b, bits, **opts)
    gpu = run_gpu(b, bits, dev, tune={"kernel": kernel}, **opts)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:], eps_hi=opts.get("eps_hi"))


@pytest.mark.parametrize("norm", ["seq", "token"])
def test_masks_c1_and_overlong(dev, norm):
    """Mask the partial-rollout (C1_MIXED) trajectories of `ragged` and, separately, the
    longest trajectories (overlong-filter stand-in); masked rows have zero gradient."""
    b = make_batch("ragged", 3)
    bits = b.logits_bits()
    masks = [_c1_mask(b), (b.lengths < np.percentile(b.lengths, 80)).astype(np.uint8)]
    assert masks[0].min() == 0 and masks[1].min() == 0
    for mask in masks:
        ref = run_oracle(b, bits, norm=norm, eps_hi=0.28, traj_mask=mask)
        gpu = run_gpu(b, bits, dev, norm=norm, eps_hi=0.28, traj_mask=mask)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:], eps_hi=0.28)
        rows = np.repeat(mask == 0, b.lengths)
        assert np.all(gpu["dlogits"][rows] == 0.0)
        assert np.all(gpu["inv_norm"][mask == 0] == 0.0)


@pytest.mark.parametrize("kernel", [1, 2])
def test_std_unbiased(dev, kernel):
    """NEXT(1) sample-std advantages (verl-style) through grpo_async_advantage_ex, with the
    DAPO options on; adv/inv_norm stay bit-exact against the oracle."""
    b = make_batch("mid32k", 4)
    bits = b.logits_bits()
    for opts in (dict(std_unbiased=True), dict(std_unbiased=True, eps_hi=0.28, norm="token")):
        ref = run_oracle(b, bits, **opts)
        gpu = run_gpu(b, bits, dev, tune={"kernel": kernel}, **opts)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:], eps_hi=opts.get("eps_hi"))
