"""-m gpu: out-of-bounds write detection without compute-sanitizer (closed on this pool,
profiles/r02_sanitizer.txt).  Every output array of every shipped kernel plan is a slice in the
middle of a larger allocation filled with a canary bit pattern; after the launches the bands
before and after each slice, and the padding columns [V, ld) of the 2-D outputs, must still
hold the canary, bit for bit."""
import numpy as np
import pytest
import torch

import paper_2604_26256_b200 as G
from paper_2604_26256_b200 import _lib as L
from synth.gen import make_batch
from tests.gpu_util import lmhead_batch, to_dev_bits

pytestmark = pytest.mark.gpu
BAND = 4096  # bytes of canary on each side


class Guarded:
    """A [*shape] tensor of `dtype` inside a canary-filled allocation."""

    def __init__(self, shape, dtype, dev, canary):
        self.n = int(np.prod(shape))
        esz = torch.empty(0, dtype=dtype).element_size()
        self.pad = BAND // esz
        self.buf = torch.empty(self.n + 2 * self.pad, dtype=dtype, device=dev)
        self.buf.view(torch.uint8).fill_(canary)
        self.t = self.buf[self.pad:self.pad + self.n].view(*shape)
        self.canary = canary

    def bands_intact(self):
        b = self.buf.view(torch.uint8).cpu().numpy()
        nb = self.pad * self.buf.element_size()
        return bool(np.all(b[:nb] == self.canary) and np.all(b[-nb:] == self.canary))


TUNES = [None, {"kernel": 2}, {"kernel": 2, "cluster_size": 2, "ctas_per_sm": 2}, {"kernel": 3},
         {"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3},
         {"kernel": 3, "chunk_kb": 16, "stages": 6, "lag": 3, "row_cache": 2, "ctas_per_sm": 256}]


@pytest.mark.parametrize("name", ["tiny", "ragged", "mid152k", "large_small"])
def test_loss_kernels_write_only_their_outputs(dev, name):
    b = make_batch(name, 2)
    bits = b.logits_bits()
    T, ld, V, N = b.T, b.ld, b.V, b.N
    lg = to_dev_bits(bits, dev)
    db = G.DeviceBatch.from_host(b, dev)
    tunes = list(TUNES) + ([{"kernel": 3, "chunk_kb": 32, "stages": 6, "lag": 3, "cluster_size": 2}]
                           if V >= 16384 else [])
    for tune in tunes:
        loss = G.GrpoAsyncLoss(tune=tune)
        adv, inv = loss.advantage(db)
        need = L.grpo_async_workspace_size(T, V, N)
        ws = Guarded((need,), torch.uint8, dev, 0xA5)
        loss._ws = ws.t
        dl = Guarded((T, ld), torch.int16, dev, 0xC3)
        outs = {k: Guarded((T,), torch.float32, dev, 0x7F) for k in ("logp", "lse", "scale")}
        ts = Guarded((N,), torch.float64, dev, 0x5A)
        st = Guarded((G.NUM_STATS,), torch.float64, dev, 0x5A)
        ts.t.zero_()
        st.t.zero_()
        half = T // 2
        for b0, b1 in ((0, half), (half, T)):
            loss.loss_chunk(lg[b0:b1], b0, b1 - b0, db.target_ids[b0:b1], db.logp_behav[b0:b1],
                            db.cu_seqlens, adv, inv, ts.t, st.t, dlogits=dl.t[b0:b1],
                            logp_out=outs["logp"].t[b0:b1], lse_out=outs["lse"].t[b0:b1],
                            scale_out=outs["scale"].t[b0:b1], V=V)
        torch.cuda.synchronize()
        for k, g in [("workspace", ws), ("dlogits", dl), ("traj_sum", ts), ("stats", st)] + list(outs.items()):
            assert g.bands_intact(), (name, tune, k)
        pad = dl.t.view(torch.uint8).cpu().numpy().reshape(T, ld * 2)[:, 2 * V:]
        assert np.all(pad == 0xC3), (name, tune, "dlogits padding columns")


@pytest.mark.parametrize("world,lag", [(2, 0), (4, 0), (2, 3), (4, 2)])
def test_vp_kernels_write_only_their_shards(dev, world, lag):
    """The vocabulary-parallel kernels -- row-wise (V = 4099), the delayed-pass-2 ring
    (152064 at R = 2, 4: one 512-thread / two 256-thread CTAs per SM; lag 2, 3 forced) and
    the look-ahead ring (262144 at R = 2) -- R ranks in one launch."""
    rng = np.random.default_rng(3)
    for V in ((4099, 152064, 262144) if lag == 0 else (152064,)):
        b = make_batch("mid152k", 3)
        import dataclasses
        b = dataclasses.replace(b, V=V, ld=(V + 7) // 8 * 8, target_ids=(b.target_ids % V).astype(np.int64))
        z = (rng.normal(size=(b.T, V)) * 2).astype(np.float32)
        from synth.gen import f32_to_bf16_bits
        bits = np.zeros((b.T, b.ld), np.uint16)
        bits[:, :V] = f32_to_bf16_bits(z)
        comm = G.VpGroup.local(world, V, b.T, dev)
        comm.lag = lag
        sc = comm.shard_cols
        lg = to_dev_bits(bits, dev)
        shards, dsh = [], []
        for q in range(world):
            sh = torch.full((b.T, sc), 0x7FC1, dtype=torch.int16, device=dev)
            lo, hi = q * sc, min((q + 1) * sc, V)
            sh[:, :hi - lo] = lg[:, lo:hi]
            shards.append(sh)
            dsh.append(Guarded((b.T, sc), torch.int16, dev, 0xC3))
        db = G.DeviceBatch.from_host(b, dev)
        loss = G.GrpoAsyncLoss()
        adv, inv = loss.advantage(db)
        ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
        st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
        loss.loss_chunk_vp(comm, shards, 0, b.T, db.target_ids, db.logp_behav, db.cu_seqlens, adv, inv,
                           ts, st, dshards=[d.t for d in dsh], V=V)
        torch.cuda.synchronize()
        for q, d in enumerate(dsh):
            assert d.bands_intact(), (V, q)
            valid = max(0, min(sc, V - q * sc))
            pad = d.t.view(torch.uint8).cpu().numpy().reshape(b.T, 2 * sc)[:, 2 * valid:]
            assert np.all(pad == 0xC3), (V, q, "shard padding")


@pytest.mark.parametrize("d", [64, 256])
def test_lmhead_kernels_write_only_their_outputs(dev, d):
    """LM head: dz (TMA-store epilogue, padding columns), dX (bf16 TMA stores), dW (TMA reduce-add)."""
    b, X, W = lmhead_batch("ragged", 5, d)
    T, V = b.T, b.V
    db = G.DeviceBatch.from_host(b, dev)
    loss = G.GrpoAsyncLoss()
    adv, inv = loss.advantage(db)
    Xd = to_dev_bits(X, dev).view(torch.bfloat16)
    Wd = to_dev_bits(W, dev).view(torch.bfloat16)
    lse = torch.empty(T, device=dev)
    scale = torch.empty(T, device=dev)
    ts = torch.zeros(b.N, dtype=torch.float64, device=dev)
    st = torch.zeros(G.NUM_STATS, dtype=torch.float64, device=dev)
    loss.lmhead_fwd(Xd, Wd, 0, T, db.target_ids, db.logp_behav, db.cu_seqlens, adv, inv, ts, st,
                    lse_out=lse, scale_out=scale)
    ld = (V + 7) // 8 * 8 + 8
    dz = Guarded((T, ld), torch.int16, dev, 0xC3)
    dX = Guarded((T, d), torch.int16, dev, 0xC3)
    dW = Guarded((V, d), torch.float32, dev, 0x00)
    for cg in (2, 1):
        L.grpo_async_lmhead_set_cta_group(cg)
        loss.lmhead_bwd(Xd, Wd, T, db.target_ids, lse, scale, dz.t.view(torch.bfloat16),
                        dhidden=dX.t.view(torch.bfloat16), dW=dW.t)
        torch.cuda.synchronize()
        for k, g in (("dz", dz), ("dX", dX), ("dW", dW)):
            assert g.bands_intact(), (cg, k)
        pad = dz.t.view(torch.uint8).cpu().numpy().reshape(T, 2 * ld)[:, 2 * V:]
        assert np.all(pad == 0xC3), (cg, "dz padding columns")
    L.grpo_async_lmhead_set_cta_group(2)
