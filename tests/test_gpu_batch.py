"""Batched objective: several parameter points per pass.

Each batched value must be bitwise its own single-point NLL, errors must be
attributed to the right point, and a fit driven through the batched objective
must follow exactly the trajectory (values, n_calls) of point-by-point calls.
"""

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def points_eval(pf, pdf, ds, params, pts):
    """(snaps, norms) per point the way the fitter builds them."""
    store = P.NormalizationStore()
    snaps, norms = [], []
    for pt in pts:
        for v, val in zip(params, pt):
            P.set_value(v, float(val))
        snap = P.snapshot(pdf.param_closure())
        snaps.append(snap)
        norms.append(P.resolve_norms(pdf, snap, store))
    return snaps, norms


def single(pf, pdf, ds, params, pt):
    for v, val in zip(params, pt):
        P.set_value(v, float(val))
    try:
        return pf.nll(pdf, ds)
    except Exception as exc:  # the batched call returns the exception in this slot
        return exc


def outcome(r):
    """Comparable form: floats bitwise, errors by type and event index."""
    if isinstance(r, Exception):
        return (type(r).__name__, getattr(r, "index", None))
    return ("ok", float(r).hex())


@pytest.mark.parametrize("config", ["c2", "c1"])
def test_batch_equals_single_bitwise(pf, config):
    rng = np.random.default_rng(4)
    n = 9 * 4096 + 777
    if config == "c2":
        (x, y), pdf, params = models.c2()
        xs = np.clip(rng.normal(5, 1, n), 0, 10)
        xs[::5000] = 0.2  # far tail: defers to the exact fix-up at the "wide tail" point below
        ds = models.dataset([x, y], [xs, np.clip(rng.exponential(2.5, n), 0, 10)])
        base = np.array([5.0, 1.0, -0.4])
    else:
        x, pdf, params = models.c1()
        xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 2), rng.exponential(3.0, n - n // 2)]), 0, 10)
        ds = models.dataset([x], [xs])
        base = np.array([5.0, 0.5, -0.3, 0.3])
    pts = [base]
    for k in range(len(base)):
        for s in (+1, -1):
            p = base.copy()
            p[k] += s * 0.01
            pts.append(p)
    # a point whose gaussian is so narrow that most events defer to the exact fix-up
    # (for the product model it underflows to zero: NonPositiveDensity, as in the reference)
    narrow = base.copy()
    narrow[1] = 0.011
    pts.append(narrow)
    if config == "c2":
        tail = base.copy()
        tail[1] = 0.1336  # u ~ -645 at x = 0.2: guard-deferred yet positive
        pts.append(tail)
    want = [outcome(single(pf, pdf, ds, params, p)) for p in pts]
    snaps, norms = points_eval(pf, pdf, ds, params, pts)
    backend = pf.DeviceBackend()
    names = tuple(sorted({o.name for node in pdf.walk() for o in node.observables}))
    cols = {k: ds.column(k) for k in names}
    got = backend.evaluate_batch(pdf, cols, snaps, norms, 0, ds.n_events)
    assert [outcome(r) for r in got] == want
    assert any(w[0] == "ok" for w in want)


@pytest.mark.parametrize("npts", [2, 8, 16])
def test_c1_points_many_blocks_per_cta_bitwise(pf, npts):
    """C1 SumPdf points (EvSum2GE::POINTS in the TMA unit kernel) over 3M
    events -- ~5 blocks per CTA, so every stage of the ring and every fold
    slot is reused while the points of a block are in flight -- each bitwise
    its single-point value (a fit-like stencil: steps of 1e-3 around a point)."""
    rng = np.random.default_rng(17)
    n = 3_000_000 + 1234
    x, pdf, params = models.c1()
    xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
    ds = models.dataset([x], [xs])
    base = np.array([4.9789, 0.5726, -0.3046, 0.3041])
    pts = [base + 1e-3 * rng.standard_normal(4) * (k > 0) for k in range(npts)]
    want = [outcome(single(pf, pdf, ds, params, p)) for p in pts]
    snaps, norms = points_eval(pf, pdf, ds, params, pts)
    cols = {"x": ds.column("x")}
    for _ in range(3):
        got = pf.DeviceBackend().evaluate_batch(pdf, cols, snaps, norms, 0, ds.n_events)
        assert [outcome(r) for r in got] == want


def test_sixteen_points_all_blocks_deferred(pf):
    """16 points (the batch maximum) over 2000 blocks where every block holds
    an event whose gaussian exponent lies in (-746, -600) at every point: all
    16 x 2000 (block, point) pairs go to the exact fix-up list at once (its
    capacity is points x blocks), and each value is still bitwise
    its own single-point NLL."""
    rng = np.random.default_rng(11)
    nb = 2000
    n = nb * 4096
    (x, y), pdf, params = models.c2()
    xs = np.clip(rng.normal(5, 0.5, n), 3, 7)  # z <= 17 elsewhere
    # z ~ 37.5 at sigma ~ 0.12: u ~ -704, past the fast path's exponent budget
    # (690 - |ln c|) yet a positive normal density in the reference
    xs[::4096] = 5.0 + 37.55 * 0.12
    ds = models.dataset([x, y], [xs, np.clip(rng.exponential(2.5, n), 0, 10)])
    pts = [np.array([5.0, 0.12 * (1.0 + 0.0002 * k), -0.4]) for k in range(16)]
    ctx = pf.device_context(0)
    want = []
    for p in pts:
        before = ctx.launch_count()
        want.append(outcome(single(pf, pdf, ds, params, p)))
        assert ctx.launch_count() - before == 2  # the pass + the fix-up of every block
    assert all(w[0] == "ok" for w in want)
    snaps, norms = points_eval(pf, pdf, ds, params, pts)
    got = pf.DeviceBackend().evaluate_batch(pdf, {"x": ds.column("x"), "y": ds.column("y")}, snaps, norms, 0,
                                            ds.n_events)
    assert [outcome(r) for r in got] == want


def test_batch_error_attributed_to_its_point(pf):
    x = P.Variable.observable("x", 0.0, 1.0)
    c0 = P.Variable("c0", 0.5, -1.0, 2.0)
    c1 = P.Variable("c1", 1.0, -2.0, 2.0)
    pdf = P.polynomial(x, [c0, c1])
    vals = np.linspace(0.0, 1.0, 9000)
    ds = models.dataset([x], [vals])
    pts = [(0.5, 1.0), (0.0, 1.0), (0.6, 1.0)]  # point 1: p(0) = 0 -> NonPositiveDensity at index 0
    snaps, norms = points_eval(pf, pdf, ds, [c0, c1], pts)
    got = pf.DeviceBackend().evaluate_batch(pdf, {"x": ds.column("x")}, snaps, norms, 0, ds.n_events)
    assert isinstance(got[1], P.errors.NonPositiveDensity) and got[1].index == 0
    assert got[0] == single(pf, pdf, ds, [c0, c1], pts[0])
    assert got[2] == single(pf, pdf, ds, [c0, c1], pts[2])


def test_batched_fit_equals_unbatched_fit(pf, golden_dir):
    """DeviceFitManager (C objective + batched stencils) == its exact
    reference-objective mode, batched or point by point == the unmodified
    reference FitManager over DeviceBackend: same n_calls, bitwise values,
    errors and minimum; the reference-objective modes also leave the
    norm-cache counters exactly where the reference's own fit leaves them."""
    import os

    g = np.load(os.path.join(golden_dir, "c2_prod.npz"))
    (x, y), pdf, params = models.c2((4.9, 1.1, -0.35))
    ds = models.dataset([x, y], [g["x"], g["y"]])
    fits = []
    for make in (lambda: pf.DeviceFitManager(pdf, ds),
                 lambda: pf.DeviceFitManager(pdf, ds, fast=False),
                 lambda: pf.DeviceFitManager(pdf, ds, batch=False, fast=False),
                 lambda: P.FitManager(pdf, ds, backend=pf.DeviceBackend())):
        for v, val in zip(params, (4.9, 1.1, -0.35)):
            P.set_value(v, val)
        fm = make()
        fits.append((fm.fit(), fm))
    (fast, fmf), (batched, fm0), (plain, fm1), (ref, fm2) = fits
    from paper_1710_08826_b200.fitting import FastObjective

    assert isinstance(fmf.objective, FastObjective)
    assert fm0.objective.batches > 0 and fm0.objective.batched_points > 10
    for other, fm in ((batched, fm0), (plain, fm1), (ref, fm2)):
        assert fast.n_calls == other.n_calls
        assert np.array_equal(fast.values, other.values)
        assert np.array_equal(fast.errors, other.errors)
        assert fast.nll_min == other.nll_min
    for fm in (fm1, fm2):
        assert fm0.store.kernel_evals == fm.store.kernel_evals
        assert fm0.store.norm_computations == fm.store.norm_computations


def test_dalitz_points_in_one_pass_bitwise(pf, golden_dir):
    """The D0 Dalitz ratio form evaluates a batch of coefficient points in one
    pass (each point's scaled coefficients in its ptv row): every value
    bitwise its own single-point NLL; a batch whose points move a mass falls
    back to one launch per point with the same result."""
    import os

    g = np.load(os.path.join(golden_dir, "c3_dalitz.npz"))
    (s12, s13), pdf, terms = models.c3(grid=(128, 128))
    ds = models.dataset([s12, s13], [g["s12"], g["s13"]])
    free = [v for t in terms for v in (t.magnitude, t.phase) if not v.fixed]
    base = np.array([v.value for v in free])
    pts = [base * (1.0 + 0.003 * k) for k in range(9)]
    want = [outcome(single(pf, pdf, ds, free, p)) for p in pts]
    snaps, norms = points_eval(pf, pdf, ds, free, pts)
    cols = {"s12": ds.column("s12"), "s13": ds.column("s13")}
    ctx = pf.device_context(0)
    b = ctx.launch_count()
    got = pf.DeviceBackend().evaluate_batch(pdf, cols, snaps, norms, 0, ds.n_events)
    assert ctx.launch_count() - b == 1  # one pass for all nine points
    assert [outcome(r) for r in got] == want
    # a floating mass: shapes differ between points -> per-point launches, same bits
    mass = terms[1].mass
    mass.fixed = False
    try:
        params = free + [mass]
        pts2 = [np.append(p, mass.value * (1.0 + 1e-4 * k)) for k, p in enumerate(pts[:4])]
        want2 = [outcome(single(pf, pdf, ds, params, p)) for p in pts2]
        snaps2, norms2 = points_eval(pf, pdf, ds, params, pts2)
        got2 = pf.DeviceBackend().evaluate_batch(pdf, cols, snaps2, norms2, 0, ds.n_events)
        assert [outcome(r) for r in got2] == want2
    finally:
        mass.fixed = True


def test_gauss_poly_points_in_one_pass_bitwise(pf):
    """ProdPdf(gaussian(x), polynomial(y)) (C2p's product evaluator) batches
    points in one pass too; every value bitwise its single-point NLL."""
    rng = np.random.default_rng(6)
    n = 30 * 4096 + 321
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    mu, sg = P.Variable("mu", 5.0, 0.0, 10.0), P.Variable("sg", 1.0, 0.1, 5.0)
    cs = [P.Variable(f"c{k}", v, -10.0, 10.0) for k, v in enumerate((1.0, 0.3, 0.05))]
    pdf = P.prod_pdf([P.gaussian(x, mu, sg), P.polynomial(y, cs)])
    ds = models.dataset([x, y], [np.clip(rng.normal(5, 1, n), 0, 10), rng.uniform(0, 10, n)])
    params = [mu, sg] + cs
    base = np.array([5.0, 1.0, 1.0, 0.3, 0.05])
    pts = [base + 0.01 * np.eye(5)[k % 5] * (1 if k < 5 else -1) for k in range(10)]
    want = [outcome(single(pf, pdf, ds, params, p)) for p in pts]
    snaps, norms = points_eval(pf, pdf, ds, params, pts)
    ctx = pf.device_context(0)
    b = ctx.launch_count()
    got = pf.DeviceBackend().evaluate_batch(pdf, {"x": ds.column("x"), "y": ds.column("y")}, snaps, norms, 0,
                                            ds.n_events)
    assert ctx.launch_count() - b == 1
    assert [outcome(r) for r in got] == want


@pytest.mark.parametrize("shape", ["poly", "expo_poly"])
def test_single_term_product_points_in_one_pass_bitwise(pf, shape):
    """EvProd1 (a lone polynomial; exponential x polynomial) batches points in
    one pass; every value bitwise its single-point NLL."""
    rng = np.random.default_rng(8)
    n = 20 * 4096 + 77
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    cs = [P.Variable(f"q{k}", v, -10.0, 10.0) for k, v in enumerate((1.0, 0.3, 0.05))]
    if shape == "poly":
        pdf, obs, params, base = P.polynomial(x, cs), [x], cs, np.array([1.0, 0.3, 0.05])
    else:
        a = P.Variable("a", -0.2, -5.0, 5.0)
        pdf, obs, params = P.prod_pdf([P.exponential(x, a), P.polynomial(y, cs)]), [x, y], [a] + cs
        base = np.array([-0.2, 1.0, 0.3, 0.05])
    cols = [rng.uniform(0, 10, n) for _ in obs]
    ds = models.dataset(obs, cols)
    pts = [base * (1.0 + 0.002 * k) for k in range(7)]
    want = [outcome(single(pf, pdf, ds, params, p)) for p in pts]
    snaps, norms = points_eval(pf, pdf, ds, params, pts)
    ctx = pf.device_context(0)
    b = ctx.launch_count()
    got = pf.DeviceBackend().evaluate_batch(pdf, {o.name: ds.column(o.name) for o in obs}, snaps, norms, 0,
                                            ds.n_events)
    assert ctx.launch_count() - b == 1
    assert [outcome(r) for r in got] == want
