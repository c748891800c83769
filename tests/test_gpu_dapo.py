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
# the row-wise kernel K3b, the production K3c instantiation (stream_kernel<512,1,2048,1>, the
# auto plan for V >= 90000) and the split-row K3c (stream_kernel<512,1,2048,2>, V >= 200000)
TUNES = {"rowwise": {"kernel": 2},
         "stream32": {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3},
         "split": {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3, "cluster_size": 2}}


def _c1_mask(b):
    v = O.validate(b.version_ids, b.cu_seqlens, b.group_ids, b.target_ids, P=b.P, V=b.V, G=b.G,
                   tbs=b.tbs, v_theta=b.v_theta, K=b.K, token_version=b.token_version)
    return ((v["traj_flags"] & (1 << 5)) == 0).astype(np.uint8)


@pytest.mark.parametrize("tune", list(TUNES))
@pytest.mark.parametrize("opts", OPTS, ids=["cliphigher", "tokenmean", "both"])
@pytest.mark.parametrize("name", ["mid32k", "mid152k", "large_small"])
def test_dapo_options(dev, tune, opts, name):
    b = make_batch(name, 2)
    bits = b.logits_bits()
    ref = run_oracle(b, bits, **opts)
    gpu = run_gpu(b, bits, dev, tune=TUNES[tune], **opts)
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
        for tune in (None, TUNES["stream32"], TUNES["split"]):
            gpu = run_gpu(b, bits, dev, norm=norm, eps_hi=0.28, traj_mask=mask, tune=tune)
            compare(gpu, ref, b, logits_pad=bits[:, b.V:], eps_hi=0.28)
            rows = np.repeat(mask == 0, b.lengths)
            assert np.all(gpu["dlogits"][rows] == 0.0)
            assert np.all(gpu["inv_norm"][mask == 0] == 0.0)


@pytest.mark.parametrize("tune", list(TUNES))
def test_std_unbiased(dev, tune):
    """NEXT(1) sample-std advantages (verl-style) through grpo_async_advantage_ex, with the
    DAPO options on; adv/inv_norm stay bit-exact against the oracle."""
    b = make_batch("mid32k", 4)
    bits = b.logits_bits()
    for opts in (dict(std_unbiased=True), dict(std_unbiased=True, eps_hi=0.28, norm="token")):
        ref = run_oracle(b, bits, **opts)
        gpu = run_gpu(b, bits, dev, tune=TUNES[tune], **opts)
        compare(gpu, ref, b, logits_pad=bits[:, b.V:], eps_hi=opts.get("eps_hi"))
