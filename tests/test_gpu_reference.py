"""The unmodified reference (parafit, baseline/_ref) driving the device engine
at BASELINE.json's sizes, against the reference's own CPU path on the SAME
arrays.

* NLL: the reference ``nll`` (P/engine.py:214-243) with ``DeviceBackend`` and
  the device norm hooks vs the reference ``nll`` with ``Backend("pool")`` and
  its own norms -- C1 at 1M, C2 at 10M, C3 at 10M events; <= 1e-10 relative.
* Fits: the reference ``FitManager`` (P/fitting.py:410-495) over
  ``DeviceBackend`` and :class:`DeviceFitManager` (batched stencils) vs the
  reference ``FitManager`` over ``Backend("pool")``; parameters within 1e-6
  relative or 1e-3 sigma, minimum within 1e-10.

Inputs are device-generated synthetic events (Philox samplers) downloaded
once; both sides read exactly those float64 columns.
"""

import os

import numpy as np
import pytest

from paper_1710_08826_b200._reference import parafit as P
from tests import models

pytestmark = pytest.mark.gpu

RTOL = 1e-10


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


@pytest.fixture(autouse=True)
def _pool_env(monkeypatch):
    # PARAFIT_WORKERS silently overrides Backend("pool", workers=...) (P/engine.py:43-47)
    monkeypatch.delenv("PARAFIT_WORKERS", raising=False)


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def pool():
    return P.Backend("pool", workers=os.cpu_count() or 1)


_DATA = {}


def data(pf, cfg, n):
    """(observables, pdf, params, dataset) of a config over device-generated events."""
    from paper_1710_08826_b200 import mcgen

    key = (cfg, n)
    if key not in _DATA:
        if cfg == "c1":
            cols = [mcgen.device_sumpdf_1d(n, 5.0, 0.5, -0.3, 0.3, 0.0, 10.0, 101)]
        elif cfg == "c2":
            cols = list(mcgen.device_prod_2d(n, 5.0, 1.0, -0.4, 0.0, 10.0, 102))
        else:
            terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
            cols = list(mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, 103))
        _DATA[key] = cols
    cols = _DATA[key]
    if cfg == "c1":
        x, pdf, params = models.c1()
        obs = [x]
    elif cfg == "c2":
        obs, pdf, params = models.c2()
    else:
        obs, pdf, rts = models.c3()
        params = [v for t in rts for v in (t.magnitude, t.phase) if not v.fixed]
    return list(obs), pdf, list(params), pf.DeviceDataSet.from_columns(list(obs), cols, device=None)


POINTS = {
    "c1": [(5.0, 0.5, -0.3, 0.3), (4.93, 0.52, -0.31, 0.27)],
    "c2": [(5.0, 1.0, -0.4), (5.06, 0.97, -0.38)],
    "c3": [(0.73, -0.03, 0.55, 0.28, 20.0, -0.5), (0.8, 0.05, 0.5, 0.3, 18.0, -0.45)],
}


@pytest.mark.parametrize("cfg,n", [("c1", 1_000_000), ("c2", 10_000_000), ("c3", 10_000_000)])
def test_reference_nll_device_backend_vs_reference_pool(pf, cfg, n):
    obs, pdf, params, ds = data(pf, cfg, n)
    backend = pf.DeviceBackend()
    for pt in POINTS[cfg]:
        for v, val in zip(params, pt):
            P.set_value(v, float(val))
        snap = P.snapshot(pdf.param_closure())
        got = P.nll(pdf, ds, snap, backend, P.NormalizationStore())  # device hooks (installed)
        with pf.reference_norms():
            want = P.nll(pdf, ds, snap, pool(), P.NormalizationStore())
            # same norms on both sides isolates the kernel + reduction
            same_norms = P.nll(pdf, ds, snap, backend, P.NormalizationStore())
        assert rel(got, want) <= RTOL, (cfg, pt, got, want)
        assert rel(same_norms, want) <= RTOL, (cfg, pt, same_norms, want)


def _check_fit(result, want):
    assert result.status == want.status == "converged"
    assert list(result.names) == list(want.names)
    for name, v, e, rv, re in zip(result.names, result.values, result.errors, want.values, want.errors):
        tol = max(1e-6 * abs(rv), 1e-3 * re)
        assert abs(v - rv) <= tol, (name, v, rv, tol)
        assert abs(e - re) <= 1e-3 * re, (name, e, re)
    assert rel(result.nll_min, want.nll_min) <= RTOL


FIT_STARTS = {
    "c1": (4.8, 0.6, -0.25, 0.35),
    "c2": (4.9, 1.1, -0.35),
    "c3": (0.8, 0.0, 0.5, 0.3, 19.0, -0.45),
}


@pytest.mark.parametrize("cfg,n", [("c1", 1_000_000), ("c2", 10_000_000), ("c3", 10_000_000)])
def test_reference_fitmanager_device_vs_reference_pool(pf, cfg, n):
    obs, pdf, params, ds = data(pf, cfg, n)

    def start():
        for v, val in zip(params, FIT_STARTS[cfg]):
            P.set_value(v, float(val))

    start()
    with pf.reference_norms():
        want = P.FitManager(pdf, ds, backend=pool()).fit()
    start()
    on_device = P.FitManager(pdf, ds, backend=pf.DeviceBackend()).fit()
    start()
    batched = pf.DeviceFitManager(pdf, ds, fast=False).fit()
    start()
    fast = pf.DeviceFitManager(pdf, ds).fit()  # the objective in C (+ batched stencils)
    _check_fit(on_device, want)
    _check_fit(batched, want)
    _check_fit(fast, want)
    # the batched stencils change nothing but the number of device passes
    assert batched.n_calls == on_device.n_calls
    assert np.array_equal(batched.values, on_device.values)
    assert batched.nll_min == on_device.nll_min
    if cfg != "c3":  # gaussian / exponential norms in C are the reference's bits
        assert fast.n_calls == on_device.n_calls and np.array_equal(fast.values, on_device.values)
