"""ProdPdf(gaussian(x), polynomial(y)) -- the C2p shape -- on its product-mode
evaluator (EvGaussPoly: log sum of the gaussian exponents, unit product of
the polynomial values, one logarithm per 16 events), and the general
single-term product evaluator (EvProd1: a lone polynomial, exponential x
polynomial, three-column products).

* every product-mode shell (pipeline 1 / 3: TMA unit kernel, 2: bulk
  prefetch) gives bitwise the same block values;
* NLL within 1e-10 of the reference ``nll`` with ``Backend("pool")`` on the
  same arrays (P/engine.py:214-243), and of the log-domain kernel (pipeline 0);
* events the evaluator cannot certify (gaussian exponent below -600, a
  polynomial value far from 1, a non-positive polynomial) defer their block
  to the literal fix-up: the value stays the reference's, the error is the
  reference's error (class, event index, density).
"""

import ctypes
import os

import numpy as np
import pytest

from paper_1710_08826_b200._reference import errors as E
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

RTOL = 1e-10
N = 2_000_000 + 1237  # ragged, odd tail


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


@pytest.fixture(autouse=True)
def _pool_env(monkeypatch):
    monkeypatch.delenv("PARAFIT_WORKERS", raising=False)


def model(coefs=(1.0, 0.3, 0.05), mu=5.0, sigma=1.0):
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    c = [P.Variable(f"c{k}", v, -10.0, 10.0, step=1e-3) for k, v in enumerate(coefs)]
    pdf = P.prod_pdf([P.gaussian(x, P.Variable("mu", mu, 0.0, 10.0), P.Variable("sigma", sigma, 0.01, 5.0)),
                      P.polynomial(y, c)])
    return (x, y), pdf


def columns(n=N, seed=11):
    rng = np.random.default_rng(seed)
    xs = np.clip(rng.normal(5.0, 1.0, n), 0.0, 10.0)
    ys = rng.uniform(0.0, 10.0, n)
    return xs, ys


def ref_nll(pf, pdf, obs, cols):
    """The reference nll, its own pool backend and norms, on the same arrays."""
    ds = pf.DeviceDataSet.from_columns(list(obs), list(cols), device=None)
    with pf.reference_norms():
        return P.nll(pdf, ds, P.snapshot(pdf.param_closure()), P.Backend("pool", workers=os.cpu_count() or 1),
                     P.NormalizationStore())


def block_sums(pf, pdf, cols):
    from paper_1710_08826_b200 import _lib as L

    ctx = pf.device_context(0)
    plan = ctx.plan_for(pdf, ("x", "y"))
    st = ctx.store_for(list(cols))
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    vals, nv = plan.pack(snap, norms)
    n = len(cols[0])
    nb = -(-n // 4096)
    out = np.empty(nb)
    err = L.PfbErr()
    L.check(L.lib().pfb_nll_block_sums(ctx.handle, plan.handle, st, 0, n, 0, L.dptr(vals), len(vals),
                                       L.dptr(nv), len(nv), L.dptr(out), nb, ctypes.byref(err)),
            "pfb_nll_block_sums")
    return out


def with_pipeline(pf, mode, fn):
    ctx = pf.device_context(0)
    ctx.set_pipeline(mode)
    try:
        return fn()
    finally:
        ctx.set_pipeline(1)


def test_product_shells_bitwise_and_reference(pf):
    obs, pdf = model()
    cols = columns()
    sums = {m: with_pipeline(pf, m, lambda: block_sums(pf, pdf, cols)) for m in (1, 2, 3)}
    assert sums[1].tobytes() == sums[2].tobytes() == sums[3].tobytes()
    ds = pf.DeviceDataSet.from_columns(list(obs), list(cols), device=None)
    got = {m: with_pipeline(pf, m, lambda: pf.nll(pdf, ds)) for m in (1, 2, 3, 0)}
    assert got[1] == got[2] == got[3]
    want = ref_nll(pf, pdf, obs, cols)
    for m, v in got.items():
        assert abs(v - want) <= RTOL * abs(want), (m, v, want)


def test_uncertified_events_take_the_fixup(pf):
    # a gaussian exponent of about -648 (z = 36: the reference's exp is still
    # normal), and a polynomial value near 2^-400 at y = 0 with c0 tiny
    obs, pdf = model(coefs=(1e-120, 1.0, 0.05), mu=9.0, sigma=0.25)
    xs, ys = columns(300_000, seed=5)
    xs = np.clip(xs + 4.0, 0.0, 10.0)
    xs[77_777] = 0.0
    ys[123_456] = 0.0
    want = ref_nll(pf, pdf, obs, (xs, ys))
    ds = pf.DeviceDataSet.from_columns(list(obs), [xs, ys], device=None)
    ctx = pf.device_context(0)
    pf.nll(pdf, ds)  # warm (norms, plan, store)
    clean = pf.DeviceDataSet.from_columns(list(obs), [np.clip(xs, 5.0, 10.0), np.maximum(ys, 1.0)], device=None)
    pf.nll(pdf, clean)
    before = ctx.launch_count()
    pf.nll(pdf, clean)
    one_pass = ctx.launch_count() - before
    before = ctx.launch_count()
    got = pf.nll(pdf, ds)
    assert ctx.launch_count() - before == one_pass + 1  # + the literal fix-up of the two blocks
    assert abs(got - want) <= RTOL * abs(want), (got, want)


def test_negative_polynomial_is_the_reference_error(pf):
    obs, pdf = model(coefs=(1.0, -0.15, 0.0))  # negative for y > 6.67
    xs, ys = columns(100_000, seed=9)
    ys = np.clip(ys, 0.0, 6.5)
    ys[54_321] = 7.5
    with pytest.raises(E.ParafitError) as ref_err:
        ref_nll(pf, pdf, obs, (xs, ys))
    ds = pf.DeviceDataSet.from_columns(list(obs), [xs, ys], device=None)
    with pytest.raises(E.ParafitError) as dev_err:
        pf.nll(pdf, ds)
    assert type(dev_err.value) is type(ref_err.value)
    assert str(dev_err.value) == str(ref_err.value)


@pytest.mark.parametrize("shape", ["poly", "expo_poly", "prod3"])
def test_single_term_products_with_a_polynomial(pf, shape):
    """EvProd1 on 1 / 2 / 3 columns: NLL within 1e-10 of the reference's own
    nll on the same 1M events, product shells bitwise (pipelines 1, 2, 3 where
    the shape has a staging kernel), the log-domain SIMT kernel (pipeline 0)
    within 1e-10."""
    rng = np.random.default_rng(17)
    n = 1_000_000 + 333
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    z = P.Variable.observable("z", 0.0, 10.0)
    poly = lambda o, cs: P.polynomial(o, [P.Variable(f"{o.name}c{k}", v, -10.0, 10.0) for k, v in enumerate(cs)])
    if shape == "poly":
        obs, pdf = [x], poly(x, (1.0, 0.2, 0.03, 0.001))
    elif shape == "expo_poly":
        obs, pdf = [x, y], P.prod_pdf([P.exponential(x, P.Variable("a", -0.2, -5.0, 5.0)), poly(y, (2.0, 0.1))])
    else:
        obs = [x, y, z]
        pdf = P.prod_pdf([P.gaussian(x, P.Variable("m", 5.0, 0.0, 10.0), P.Variable("s", 1.5, 0.1, 5.0)),
                          P.exponential(y, P.Variable("a", 0.1, -5.0, 5.0)), poly(z, (0.5, 1.0, 0.2))])
    cols = [np.clip(rng.normal(5.0, 2.0, n), 0.0, 10.0) for _ in obs]
    ds = pf.DeviceDataSet.from_columns(obs, cols, device=None)
    want = ref_nll(pf, pdf, obs, cols)
    got = {m: with_pipeline(pf, m, lambda: pf.nll(pdf, ds)) for m in (1, 2, 3, 0)}
    if len(obs) <= 2:
        assert got[1] == got[2] == got[3]
    for m, v in got.items():
        assert abs(v - want) <= RTOL * abs(want), (shape, m, v, want)
