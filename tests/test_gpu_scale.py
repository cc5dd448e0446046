"""Large event counts: 64-bit indexing end to end.  One NLL over 600M C2
events (9.6 GB of columns in HBM) equals, bit for bit, the exact sum of the
block sums of its block-aligned pieces, and an error index beyond 2^31 is
reported exactly."""

import ctypes

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

N = 600_000_000


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def test_600m_events_whole_equals_pieces(pf):
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen, sharding

    ctx = pf.device_context(0)
    st = mcgen._device_store(ctx, 2, N)
    L.check(L.lib().pfb_gen_1d(ctx.handle, 1, 5.0, 1.0, -0.4, 0.0, 0.0, 10.0, 77, N, st), "pfb_gen_1d")
    (x, y), pdf, _ = models.c2()
    plan = ctx.plan_for(pdf, ("x", "y"))
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    vals, nv = plan.pack(snap, norms)
    out, err = ctypes.c_double(), L.PfbErr()
    L.check(L.lib().pfb_nll(ctx.handle, plan.handle, st, 0, N, 0, L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                            ctypes.byref(out), ctypes.byref(err)), "pfb_nll")
    whole = out.value
    # block-aligned pieces through the block-sum export, summed exactly on the host
    bounds = [0, 150_003_712, 300_007_424, 450_011_136, N]  # multiples of 4096
    acc = np.zeros(L.PFB_ACC_WORDS, dtype=np.int64)
    for a, b in zip(bounds[:-1], bounds[1:]):
        nb = -(-(b - a) // 4096)
        bs = np.empty(nb)
        L.check(L.lib().pfb_nll_block_sums(ctx.handle, plan.handle, st, a, b, a, L.dptr(vals), len(vals),
                                           L.dptr(nv), len(nv), L.dptr(bs), nb, ctypes.byref(err)),
                "pfb_nll_block_sums")
        acc += sharding.acc_of_values(bs)
    assert sharding.round_acc(acc) == whole
    assert np.isfinite(whole) and whole > 0
    L.lib().pfb_store_destroy(st)


def test_error_index_beyond_2_31(pf):
    """NonPositiveDensity at global event 2^31 + 12345 of a 2.3e9-event range
    addressed through an index offset (the shard path)."""
    from paper_1710_08826_b200._reference import errors as E

    x = P.Variable.observable("x", 0.0, 1.0)
    pdf = P.polynomial(x, [P.Variable("c0", 0.5, -1.0, 2.0), P.Variable("c1", 1.0, -2.0, 2.0)])
    vals = np.linspace(0.0, 1.0, 100_000)
    ds = models.dataset([x], [vals])
    backend = pf.DeviceBackend()
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    P.set_value(pdf.parameters[0], 0.0)  # p(0) = 0 at local event 0
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    off = (1 << 31) + 12345
    with pytest.raises(E.NonPositiveDensity) as ei:
        backend.evaluate(pdf, {"x": ds.column("x")}, snap, norms, 0, ds.n_events, index_offset=off)
    assert ei.value.index == off


def test_batched_points_at_scale_equal_single(pf):
    """The in-kernel batched objective over 200M events (4 points per pass)
    gives each point's single-call NLL bit for bit."""
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen

    n = 200_000_000
    ctx = pf.device_context(0)
    st = mcgen._device_store(ctx, 2, n)
    L.check(L.lib().pfb_gen_1d(ctx.handle, 1, 5.0, 1.0, -0.4, 0.0, 0.0, 10.0, 78, n, st), "pfb_gen_1d")
    (x, y), pdf, params = models.c2()
    plan = ctx.plan_for(pdf, ("x", "y"))
    store = P.NormalizationStore()
    snaps, norms = [], []
    for k in range(4):
        P.set_value(params[0], 5.0 + 0.01 * k)
        P.set_value(params[1], 1.0 - 0.005 * k)
        snap = P.snapshot(pdf.param_closure())
        snaps.append(snap)
        norms.append(P.resolve_norms(pdf, snap, store))
    vals, nv = plan.pack_batch(snaps, norms)
    out = np.empty(4)
    errs = (L.PfbErr * 4)()
    L.check(L.lib().pfb_nll_batch(ctx.handle, plan.handle, st, 0, n, 0, L.dptr(vals), 4, vals.shape[1],
                                  L.dptr(nv), nv.shape[1], L.dptr(out), errs), "pfb_nll_batch")
    for k in range(4):
        v1, n1 = plan.pack(snaps[k], norms[k])
        single, err = ctypes.c_double(), L.PfbErr()
        L.check(L.lib().pfb_nll(ctx.handle, plan.handle, st, 0, n, 0, L.dptr(v1), len(v1), L.dptr(n1), len(n1),
                                ctypes.byref(single), ctypes.byref(err)), "pfb_nll")
        assert out[k] == single.value, k
    L.lib().pfb_store_destroy(st)


def test_dalitz_100m_product_kernel_matches_reference_tree_kernel(pf):
    """C4 scale: the TMA product kernel (ratio evaluator) and the SIMT
    reference-tree kernel agree to rounding on 100M Dalitz events."""
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen

    terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
    s12, s13 = mcgen.device_dalitz(100_000_000, terms, models.D_CHANNEL_T, 4)
    (o12, o13), pdf, _ = models.c3()
    ds = pf.DeviceDataSet.from_columns([o12, o13], [s12, s13], device=None)
    ctx = pf.device_context(0)
    fast = pf.nll(pdf, ds)
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, 0), "pfb_ctx_set_pipeline")
    try:
        ref = pf.nll(pdf, ds)
    finally:
        L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, 1), "pfb_ctx_set_pipeline")
    assert abs(fast - ref) <= 1e-12 * abs(ref)
