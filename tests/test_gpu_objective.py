"""The minimiser's objective in C (pfb_objective, fitting.FastObjective)
against the reference objective (FitManager.fcn, P/fitting.py:436-447).

* gaussian / exponential / add / prod models: every value bitwise the
  reference objective's (same raw values, the reference's norm formulas on
  the same doubles through libm), so whole fits are bitwise identical;
* Dalitz (fixed shapes): norm from the fixed overlap matrix, NLL within
  1e-12 of the reference objective's; fit within the north-star tolerance;
* failures take the reference path: out-of-bounds x -> OutOfBounds, a
  non-positive norm -> NonPositiveNorm, fractions -> FractionOutOfRange;
* models it cannot express (free polynomial coefficients) fall back to the
  reference objective.
"""

import math

import numpy as np
import pytest

from paper_1710_08826_b200._reference import errors as E
from paper_1710_08826_b200._reference import parafit as P
from tests import models

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def _c1_data(n, seed=3):
    rng = np.random.default_rng(seed)
    x, pdf, params = models.c1()
    xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
    return x, pdf, params, models.dataset([x], [xs])


def test_values_bitwise_reference_objective(pf):
    from paper_1710_08826_b200.fitting import FastObjective

    x, pdf, params, ds = _c1_data(40 * 4096 + 77)
    fast = pf.DeviceFitManager(pdf, ds).fcn()
    exact = pf.DeviceFitManager(pdf, ds, fast=False).fcn()
    assert isinstance(fast._objective, FastObjective)
    rng = np.random.default_rng(1)
    for _ in range(50):
        pt = np.array([rng.uniform(4.5, 5.5), rng.uniform(0.3, 0.8), rng.uniform(-0.5, -0.1), rng.uniform(0.1, 0.6)])
        assert fast(pt) == exact(pt)
    assert fast.n_calls == exact.n_calls == 50


def test_fit_bitwise_reference_fitmanager(pf):
    x, pdf, params, ds = _c1_data(100 * 4096 + 5)
    start = (4.8, 0.6, -0.25, 0.35)
    res = []
    for make in (lambda: pf.DeviceFitManager(pdf, ds), lambda: P.FitManager(pdf, ds, backend=pf.DeviceBackend())):
        for v, val in zip(params, start):
            P.set_value(v, val)
        res.append(make().fit())
    fast, ref = res
    assert fast.status == ref.status == "converged"
    assert fast.n_calls == ref.n_calls
    assert np.array_equal(fast.values, ref.values) and np.array_equal(fast.errors, ref.errors)
    assert fast.nll_min == ref.nll_min
    # write-back as the reference FitManager does
    assert [v.value for v in params] == list(fast.values)


def test_dalitz_fast_objective_matches_reference(pf, golden_dir):
    import os

    from paper_1710_08826_b200.fitting import FastObjective

    g = np.load(os.path.join(golden_dir, "c3_dalitz.npz"))
    (s12, s13), pdf, terms = models.c3(grid=(128, 128))
    ds = models.dataset([s12, s13], [g["s12"], g["s13"]])
    free = [v for t in terms for v in (t.magnitude, t.phase) if not v.fixed]
    fast = pf.DeviceFitManager(pdf, ds).fcn()
    exact = pf.DeviceFitManager(pdf, ds, fast=False).fcn()
    assert isinstance(fast._objective, FastObjective)
    base = np.array([v.value for v in free])
    for k in range(8):
        pt = base * (1.0 + 0.01 * k)
        a, b = fast(pt), exact(pt)
        assert abs(a - b) <= 1e-12 * abs(b), (k, a, b)
    start = [0.8, 0.0, 0.5, 0.3, 19.0, -0.45]
    fits = []
    for make in (lambda: pf.DeviceFitManager(pdf, ds), lambda: pf.DeviceFitManager(pdf, ds, fast=False)):
        for v, val in zip(free, start):
            P.set_value(v, val)
        fits.append(make().fit())
    f, r = fits
    assert f.status == r.status == "converged"
    for v, e, rv, re in zip(f.values, f.errors, r.values, r.errors):
        assert abs(v - rv) <= max(1e-6 * abs(rv), 1e-3 * re)
    assert abs(f.nll_min - r.nll_min) <= 1e-10 * abs(r.nll_min)


def test_failures_take_the_reference_path(pf):
    x, pdf, params, ds = _c1_data(9 * 4096 + 1)
    fcn = pf.DeviceFitManager(pdf, ds).fcn()
    with pytest.raises(E.OutOfBounds):
        fcn(np.array([5.0, 0.5, -0.3, 1.5]))  # f outside [0, 1]
    with pytest.raises(E.OutOfBounds):
        fcn(np.array([5.0, math.nan, -0.3, 0.3]))
    # a sum whose fractions leave a negative remainder: FractionOutOfRange
    y = P.Variable.observable("y", 0.0, 10.0)
    f1, f2 = P.Variable("f1", 0.3, 0.0, 1.0), P.Variable("f2", 0.3, 0.0, 1.0)
    tree = P.add_pdf([P.gaussian(y, P.Variable("m", 5.0, fixed=True), P.Variable("s", 2.0, fixed=True)),
                      P.exponential(y, P.Variable("a", -0.1, fixed=True)),
                      P.gaussian(y, P.Variable("m2", 3.0, fixed=True), P.Variable("s2", 3.0, fixed=True))], [f1, f2])
    dsy = models.dataset([y], [ds.column("x")])
    fcn2 = pf.DeviceFitManager(tree, dsy).fcn()
    assert math.isfinite(fcn2(np.array([0.3, 0.3])))
    with pytest.raises(E.FractionOutOfRange):
        fcn2(np.array([0.7, 0.6]))
    # a gaussian whose sigma may reach 0: NonPositiveNorm from the reference path
    z = P.Variable.observable("z", 0.0, 1.0)
    sg = P.Variable("sg", 0.2, 0.0, 1.0)
    node = P.gaussian(z, P.Variable("mz", 0.5, 0.0, 1.0), sg)
    dsz = models.dataset([z], [np.linspace(0.01, 0.99, 5000)])
    fcn3 = pf.DeviceFitManager(node, dsz).fcn()
    assert math.isfinite(fcn3(np.array([0.5, 0.2])))
    with pytest.raises(E.NonPositiveNorm):
        fcn3(np.array([0.5, 0.0]))


def test_polynomial_norm_in_c_and_fallback(pf):
    """Free polynomial coefficients: the device GL integral launched from C
    (PFB_NORM_QUADRATURE) -- the same kernel the reference-path hook runs, so
    the values are bitwise; a model with a custom norm hook (grid-mode
    gaussian) falls back to the reference objective."""
    from paper_1710_08826_b200.fitting import DeviceObjective, FastObjective

    x = P.Variable.observable("x", 0.0, 1.0)
    node = P.polynomial(x, [P.Variable("c0", 1.0, 0.1, 2.0), P.Variable("c1", 0.2, -0.5, 0.5),
                            P.Variable("c2", 0.1, 0.0, 1.0)])
    ds = models.dataset([x], [np.linspace(0.0, 1.0, 30001)])
    fast = pf.DeviceFitManager(node, ds).fcn()
    exact = pf.DeviceFitManager(node, ds, fast=False).fcn()
    assert isinstance(fast._objective, FastObjective)
    rng = np.random.default_rng(3)
    for _ in range(20):
        pt = np.array([rng.uniform(0.5, 1.5), rng.uniform(-0.3, 0.3), rng.uniform(0.0, 0.5)])
        assert fast(pt) == exact(pt)
    # a coefficient move that makes the density dip negative inside the box:
    # NegativeDensity from the GL abscissas (the reference path), or from the events
    with pytest.raises((E.NegativeDensity, E.NonPositiveDensity)):
        fast(np.array([0.1, -0.5, 0.0]))
    start = (1.0, 0.2, 0.1)
    fits = []
    for make in (lambda: pf.DeviceFitManager(node, ds), lambda: pf.DeviceFitManager(node, ds, fast=False)):
        for v, val in zip(node.parameters, start):
            P.set_value(v, val)
        fits.append(make().fit())
    assert fits[0].n_calls == fits[1].n_calls and np.array_equal(fits[0].values, fits[1].values)
    with pf.device_norms(grid_kinds=("gaussian",)):
        g = P.gaussian(x, P.Variable("gm", 0.5, 0.0, 1.0), P.Variable("gs", 0.3, 0.05, 1.0))
        fcn = pf.DeviceFitManager(g, ds).fcn()
        assert type(fcn._objective) is DeviceObjective and not isinstance(fcn._objective, FastObjective)
        assert math.isfinite(fcn(np.array([0.5, 0.3])))


def test_batched_quadrature_norms_equal_sequential(pf):
    """pfb_objective_eval_batch enqueues every quadrature norm of its points
    into separate result slots and waits once (flushing when the 16 slots run
    out); the values must be the sequential objective's bit for bit, norms
    reused from the previous point included, and a quadrature that fails
    mid-batch (NegativeDensity at a GL abscissa) must end the list where the
    sequential calls end it, with the same exception."""
    from paper_1710_08826_b200.fitting import FastObjective

    x = P.Variable.observable("x", 0.0, 1.0)
    p1 = P.polynomial(x, [P.Variable("a0", 1.0, 0.01, 2.0), P.Variable("a1", 0.2, -1.0, 1.0)])
    p2 = P.polynomial(x, [P.Variable("b0", 0.5, 0.01, 2.0), P.Variable("b1", 0.1, -1.0, 1.0),
                          P.Variable("b2", 0.3, 0.0, 1.0)])
    pdf = P.add_pdf([p1, p2], [P.Variable("f", 0.4, 0.0, 1.0)])
    ds = models.dataset([x], [np.random.default_rng(5).uniform(0.0, 1.0, 50_001)])
    fcn = pf.DeviceFitManager(pdf, ds).fcn()
    obj = fcn._objective
    assert isinstance(obj, FastObjective)
    rng = np.random.default_rng(11)
    base = np.array([1.0, 0.2, 0.5, 0.1, 0.3, 0.4])  # a0 a1 b0 b1 b2 f (free-parameter order below)
    names = [v.name for v in obj.free]
    assert sorted(names) == sorted(["a0", "a1", "b0", "b1", "b2", "f"])
    order = [["a0", "a1", "b0", "b1", "b2", "f"].index(n) for n in names]

    def pts(k, bad=None):
        out = []
        for j in range(k):
            pt = base.copy()
            if j % 3 == 1:
                pt[5] = rng.uniform(0.1, 0.9)  # only the fraction moves: both norms reused
            elif j % 3 == 2:
                pt[0], pt[1] = rng.uniform(0.5, 1.5), rng.uniform(-0.3, 0.3)  # one quadrature
            else:
                pt[:5] = [rng.uniform(0.5, 1.5), rng.uniform(-0.3, 0.3), rng.uniform(0.5, 1.5),
                          rng.uniform(-0.3, 0.3), rng.uniform(0.0, 0.5)]  # two
            if j == bad:
                pt[2], pt[3], pt[4] = 0.02, -0.9, 0.0  # b(x) < 0 for x > 0.022: the GL integral fails
            out.append(pt[order])
        return out

    def sequential(xs):
        out = []
        for pt in xs:
            v = obj._try(lambda pt=pt: obj._direct(pt))
            out.append(v)
            if isinstance(v, BaseException):
                break
        return out

    for k, bad in ((16, None), (16, 9), (5, 0), (16, 15), (12, 4)):
        xs = pts(k, bad)
        got = obj.evaluate_points(xs)
        want = sequential(xs)
        assert len(got) == len(want), (k, bad)
        for g, w in zip(got, want):
            if isinstance(w, BaseException):
                assert type(g) is type(w), (k, bad, g, w)
            else:
                assert g == w, (k, bad, g, w)
