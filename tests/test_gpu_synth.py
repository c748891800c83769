"""-m gpu, T1: the device twin of the input generator (synth/csrc/synth_fill.cu) against the
host generator (synth/gen.py LogitsSpec) bit for bit.  The full-size tests and bench.py fill
their logits on the device and the oracle reads the host's; these tests are what lets the
two sides meet on the same inputs.  Covered: every BASELINE config's recipe (tiny's i.i.d.
rows, the Zipf base rows of dapo / stale / prod / large), the periodic chunk (logical row
t = physical row t mod period), a row offset, and ld padding (filled with the NaN marker 0x7FC1, never read by the loss)."""
import numpy as np
import pytest
import torch

import synth.gpu as SG
from synth.gen import make_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,period", [("tiny", None), ("ragged", None), ("dapo", 4096),
                                         ("stale", 4096), ("prod", 131072), ("large", 2048)])
def test_device_fill_matches_host_bitwise(dev, name, period):
    b = make_batch(name, 1, period=period)
    V, ld = b.V, b.ld
    rng = np.random.default_rng(7)
    n = min(b.T, 384)
    for row_begin in (0, int(rng.integers(0, max(b.T - n, 1)))):
        out = torch.full((n, ld), 0x7FC5, dtype=torch.int16, device=dev)
        SG.fill_logits(out, b.logits, row_begin, n, V)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint16)
        rows = np.arange(row_begin, row_begin + n, dtype=np.int64)
        ref = b.logits.rows_bits(rows)
        assert np.array_equal(got[:, :V], ref), (name, row_begin, int((got[:, :V] != ref).sum()))
        assert np.all(got[:, V:] == np.uint16(0x7FC1))   # padding: the fill's NaN marker
    if period is not None:  # logical rows past the period repeat the physical ones
        out = torch.empty((4, ld), dtype=torch.int16, device=dev)
        SG.fill_logits(out, b.logits, period + 3, 4, V)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint16)[:, :V],
                              b.logits.rows_bits(np.arange(3, 7, dtype=np.int64)))
