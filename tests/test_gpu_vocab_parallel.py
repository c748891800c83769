"""-m gpu: NEXT(3) -- the fused loss over vocabulary-parallel logits
(grpo_async_loss_fwd_vp, Megatron-style LM-head sharding) against the
fp64 oracle on the unsharded row.  All ranks of the group run in one cooperative
launch on one GPU (the same peer-memory exchange protocol as on R GPUs); the 2-GPU
NVLink run is scripts/vp_multi_gpu.py."""
import numpy as np
import pytest

from synth.gen import make_batch
from tests.gpu_util import compare, run_gpu_vp, run_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["tiny", "mid32k", "mid152k", "ragged"])
def test_vp_parity(dev, name, world):
    b = make_batch(name, 5)
    bits = b.logits_bits()
    ref = run_oracle(b, bits)
    gpu = run_gpu_vp(b, bits, dev, world)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    assert gpu["shard_pad_untouched"]


@pytest.mark.parametrize("world", [2, 4])
def test_vp_schedules_match_bitwise(dev, world):
    """The immediate wait (lag 0, default), the deferred wait (lag 1), static and dynamic
    row assignment, and the ring kernel with pass 2 delayed by 1-3 rows (lag 2-4, plan
    kernel 9) combine the same partials in the same order: identical
    per-row outputs and dlogits, bit for bit (traj_sum / J are fp64 sums whose order
    follows the segment reduce, not the schedule)."""
    b = make_batch("mid32k", 9)
    bits = b.logits_bits()
    ref = run_gpu_vp(b, bits, dev, world, lag=0, dynamic_rows=0)
    for lag, dyn in ((1, 0), (0, 1), (1, 1), (2, 0), (3, 0), (4, 0)):
        g = run_gpu_vp(b, bits, dev, world, lag=lag, dynamic_rows=dyn)
        for k in ("logp", "lse", "scale", "traj_sum", "stats", "dlogits_raw"):
            assert np.array_equal(g[k], ref[k], equal_nan=True), (k, lag, dyn)


def test_vp_chunks_and_epochs(dev):
    """Several row chunks and repeated calls on the same exchange buffers (counters are
    never reset: call e waits for (e+1)*R arrivals)."""
    b = make_batch("mid32k", 6)
    bits = b.logits_bits()
    ref = run_oracle(b, bits)
    gpu = run_gpu_vp(b, bits, dev, 4, chunks=3, calls=3)
    assert gpu["epoch"] == 9
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("opts", [dict(eps_hi=0.28, norm="token")])
def test_vp_dapo(dev, opts):
    b = make_batch("ragged", 7)
    bits = b.logits_bits()
    mask = (b.lengths < np.percentile(b.lengths, 80)).astype(np.uint8)
    ref = run_oracle(b, bits, traj_mask=mask, **opts)
    gpu = run_gpu_vp(b, bits, dev, 2, traj_mask=mask, **opts)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:], eps_hi=opts["eps_hi"])


def test_vp_forward_only_and_empty_shards(dev):
    """dlogits NULL (forward only), and shard_cols = 512 over V = 1024 with world 4:
    shards 2 and 3 hold no column (their partial is (-inf, 0)) yet take part in the
    exchange."""
    b = make_batch("tiny", 8)
    bits = b.logits_bits()
    ref = run_oracle(b, bits, want_dlogits=False)
    gpu = run_gpu_vp(b, bits, dev, 8, want_dlogits=False)
    compare(gpu, ref, b, check_dlogits=False)
    ref = run_oracle(b, bits)
    gpu = run_gpu_vp(b, bits, dev, 4, shard_cols=512)
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])


@pytest.mark.parametrize("seed", range(8))
def test_vp_random_shapes(dev, seed):
    """Fuzz: random vocabulary, group size 1-8, shard width (incl. empty trailing shards),
    chunking and schedule, against the oracle."""
    from tests.test_gpu_parity import _adversarial_batch
    rng = np.random.default_rng(500 + seed)
    V = int(rng.choice([int(rng.integers(8, 2000)), int(rng.integers(2000, 80000))]))
    world = int(rng.integers(1, 9))
    n = int(rng.integers(4, 40))
    rows = [(rng.normal(size=V) * float(rng.uniform(0.5, 3)), int(rng.integers(0, V))) for _ in range(n)]
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    base = -(-V // (world * 8)) * 8
    sc = base if rng.integers(0, 2) else base + 8 * int(rng.integers(1, 64))
    lag = int(rng.integers(0, 5))
    gpu = run_gpu_vp(b, bits, dev, world, chunks=int(rng.integers(1, 3)), shard_cols=sc,
                     lag=lag, dynamic_rows=int(rng.integers(0, 2)) if lag < 2 else 0,
                     calls=int(rng.integers(1, 3)))
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    assert gpu["shard_pad_untouched"]


@pytest.mark.parametrize("world", [1, 2, 4])
def test_vp_stream_kernel(dev, world):
    """Long shards (>= 90000 columns) with the default schedule run the streamed ring
    kernel (plan kernel 8, loss_vp.cu vp_stream_kernel): several chunks and calls on the
    same exchange buffers, forward-only, and against the row-wise VP kernel (lag 1)."""
    import paper_2604_26256_b200 as Gp
    rng = np.random.default_rng(70 + world)
    V = {1: 100000, 2: 262144, 4: 400000}[world]  # shards >= 90000 columns
    rows = [(rng.normal(size=V) * float(rng.uniform(0.5, 3)), int(rng.integers(0, V))) for _ in range(24)]
    from tests.test_gpu_parity import _adversarial_batch
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    gpu = run_gpu_vp(b, bits, dev, world, chunks=2, calls=2)
    plan = Gp.grpo_async_last_plan()
    assert plan["kernel"] == 8, plan
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    assert gpu["shard_pad_untouched"]
    old = run_gpu_vp(b, bits, dev, world, lag=1)
    assert Gp.grpo_async_last_plan()["kernel"] == 7
    compare(old, ref, b, logits_pad=bits[:, b.V:])
    assert np.max(np.abs(old["logp"] - gpu["logp"])) < 1e-5
    ref_f = run_oracle(b, bits, want_dlogits=False)
    compare(run_gpu_vp(b, bits, dev, world, want_dlogits=False), ref_f, b, check_dlogits=False)


@pytest.mark.parametrize("V,sc,kernel", [(80000, 64000, 9), (100000, 96000, 8)])
def test_vp_stream_kernel_empty_shards(dev, V, sc, kernel):
    """shard_cols = 64000 over V = 80000 (the delayed-pass-2 ring) and 96000 over 100000 (the
    look-ahead ring) with world 4: ranks 2 and 3 hold no column (no chunk to stream; their
    partial is (-inf, 0)) yet take part in the exchange."""
    import paper_2604_26256_b200 as Gp
    from tests.test_gpu_parity import _adversarial_batch
    rng = np.random.default_rng(81)
    rows = [(rng.normal(size=V) * 2.0, int(rng.integers(0, V))) for _ in range(12)]
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    gpu = run_gpu_vp(b, bits, dev, 4, shard_cols=sc)
    assert Gp.grpo_async_last_plan()["kernel"] == kernel
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    assert gpu["shard_pad_untouched"]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("lag", [2, 3, 4])
def test_vp_delay_kernel(dev, world, lag):
    """The ring kernel with pass 2 delayed by lag - 1 rows (plan kernel 9): R = 4 shards of a
    152064 vocabulary (74 KB rows, the shape it is for) and R = 2 of 262144 (the 512-thread
    geometry), several chunks and repeated calls on the same exchange buffers, against the
    oracle; forward-only too; fewer rows per CTA than the delay (the drain-only path)."""
    import paper_2604_26256_b200 as Gp
    from tests.test_gpu_parity import _adversarial_batch
    rng = np.random.default_rng(90 + world + lag)
    V = {2: 262144, 4: 152064}[world]
    rows = [(rng.normal(size=V) * float(rng.uniform(0.5, 3)), int(rng.integers(0, V))) for _ in range(20)]
    b, bits = _adversarial_batch(V, rows)
    ref = run_oracle(b, bits)
    gpu = run_gpu_vp(b, bits, dev, world, chunks=2, calls=2, lag=lag)
    assert Gp.grpo_async_last_plan()["kernel"] == 9
    compare(gpu, ref, b, logits_pad=bits[:, b.V:])
    assert gpu["shard_pad_untouched"]
    ref_f = run_oracle(b, bits, want_dlogits=False)
    compare(run_gpu_vp(b, bits, dev, world, want_dlogits=False, lag=lag), ref_f, b, check_dlogits=False)


def test_vp_auto_plan_by_shard_width(dev):
    """The default schedule's kernel by shard width (loss_vp.cu launch_vp): >= 90000 columns
    the look-ahead ring (8), 16384..89999 the ring with pass 2 delayed by a row (9: one
    512-thread CTA per SM from 60000 columns, two 256-thread CTAs below), narrower the
    row-wise kernel (7); each against the oracle."""
    import paper_2604_26256_b200 as Gp
    for name, world, kernel in (("large_small", 2, 8), ("mid152k", 2, 9), ("mid152k", 4, 9),
                                ("mid152k", 8, 9), ("mid32k", 4, 7)):
        b = make_batch(name, 11)
        bits = b.logits_bits()
        gpu = run_gpu_vp(b, bits, dev, world)
        assert Gp.grpo_async_last_plan()["kernel"] == kernel, (name, world)
        compare(gpu, run_oracle(b, bits), b, logits_pad=bits[:, b.V:])
