"""The two kernels behind pipeline 1's log-domain unit sums -- the
register-window SIMT kernel (up to 8 blocks per SM) and the TMA-fed unit
kernel (above) -- compute the same canonical blocks: their per-block values
are bitwise equal, so an NLL does not depend on which one ran (or on how a
range was split into calls).  The whole range below is past the SIMT
threshold, each piece is below it; the last block is ragged and odd."""

import ctypes

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

N = 6_000_000 + 1235
BOUNDS = [0, 489 * 4096, 978 * 4096, N]  # block-aligned pieces of ~2M events


def block_sums(pf, L, ctx, plan, st, vals, nv, a, b):
    nb = -(-(b - a) // 4096)
    out = np.empty(nb)
    err = L.PfbErr()
    L.check(L.lib().pfb_nll_block_sums(ctx.handle, plan.handle, st, a, b, a, L.dptr(vals), len(vals),
                                       L.dptr(nv), len(nv), L.dptr(out), nb, ctypes.byref(err)),
            "pfb_nll_block_sums")
    return out


def test_simt_and_tma_unit_sums_are_bitwise_equal():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen

    ctx = pf.device_context(0)
    assert N // 4096 + 1 > 8 * 148 and max(b - a for a, b in zip(BOUNDS, BOUNDS[1:])) // 4096 + 1 <= 8 * 148
    cx, cy = mcgen.device_prod_2d(N, 5.0, 1.0, -0.4, 0.0, 10.0, 5)
    (x, y), pdf, _ = models.c2((4.97, 1.02, -0.41))
    plan = ctx.plan_for(pdf, ("x", "y"))
    st = ctx.store_for([cx, cy])
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    vals, nv = plan.pack(snap, norms)
    whole = block_sums(pf, L, ctx, plan, st, vals, nv, 0, N)
    pieces = np.concatenate([block_sums(pf, L, ctx, plan, st, vals, nv, a, b)
                             for a, b in zip(BOUNDS[:-1], BOUNDS[1:])])
    assert whole.shape == pieces.shape
    assert whole.tobytes() == pieces.tobytes()
    # and the NLL of the whole equals the exact sum of the pieces' NLL partials
    ds = pf.DeviceDataSet.from_columns([x, y], [cx, cy], device=None)
    total = pf.nll(pdf, ds)
    from paper_1710_08826_b200 import sharding

    assert sharding.round_acc(sharding.acc_of_values(pieces)) == total
