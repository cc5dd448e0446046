"""Known-answer checks of the reference's own engine tests (SURVEY 8(c):
T/test_engine.py:32-61,68-76), restated and run with the device as the
backend of the reference's ``nll``:

* one event of a standard gaussian on an unbounded observable: NLL = ln sqrt(2 pi);
* an event replicated n times scales the NLL by n (1e-13);
* a 100k-event truncated gaussian against a from-scratch per-event left fold
  (1e-9);
* a density that is exactly zero at one event reports that event's global
  index (NonPositiveDensity);
* an empty dataset raises EmptyDataSet.
"""

import math

import numpy as np
import pytest

from paper_1710_08826_b200._reference import errors as E
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def standard_gaussian():
    x = P.Variable.observable("x")  # (-inf, inf)
    return x, P.gaussian(x, P.Variable("mu", 0.0, fixed=True), P.Variable("sigma", 1.0, fixed=True))


def test_single_event_standard_gaussian(pf):
    x, node = standard_gaussian()
    ds = pf.DeviceDataSet.from_columns([x], [np.array([0.0])], device=None)
    got = P.nll(node, ds, backend=pf.DeviceBackend())
    assert abs(got - 0.5 * math.log(2.0 * math.pi)) <= 1e-12


def test_replicated_event_scales_linearly(pf):
    x, node = standard_gaussian()
    be = pf.DeviceBackend()
    single = P.nll(node, pf.DeviceDataSet.from_columns([x], [np.array([0.3])], device=None), backend=be)
    n = 1000
    rep = P.nll(node, pf.DeviceDataSet.from_columns([x], [np.full(n, 0.3)], device=None), backend=be)
    assert rep == pytest.approx(n * single, rel=1e-13)


def test_matches_naive_sequential_fold(pf):
    mu, sigma, lo, hi = 0.5, 0.1, 0.0, 1.0
    data = np.clip(np.random.default_rng(42).normal(mu, sigma, 100_000), lo, hi)
    x = P.Variable.observable("x", lo, hi)
    node = P.gaussian(x, P.Variable("mu", mu, fixed=True), P.Variable("sigma", sigma, fixed=True))
    got = P.nll(node, pf.DeviceDataSet.from_columns([x], [data], device=None), backend=pf.DeviceBackend())
    z_hi = (hi - mu) / (sigma * math.sqrt(2.0))
    z_lo = (lo - mu) / (sigma * math.sqrt(2.0))
    norm = sigma * math.sqrt(math.pi / 2.0) * (math.erf(z_hi) - math.erf(z_lo))
    total = 0.0
    for v in data:
        total += -math.log(math.exp(-0.5 * ((v - mu) / sigma) ** 2) / norm)
    assert abs(got - total) <= 1e-9 * abs(total)


def test_zero_density_reports_the_global_index(pf):
    x = P.Variable.observable("x", 0.0, 1.0)
    node = P.polynomial(x, [P.Variable("c0", 0.0, fixed=True), P.Variable("c1", 1.0, fixed=True)])  # p(x) = x
    values = np.full(5000, 0.5)
    values[4321] = 0.0
    with pytest.raises(E.NonPositiveDensity) as err:
        P.nll(node, pf.DeviceDataSet.from_columns([x], [values], device=None), backend=pf.DeviceBackend())
    assert err.value.index == 4321


def test_empty_dataset(pf):
    x, node = standard_gaussian()
    with pytest.raises(E.EmptyDataSet):
        P.nll(node, P.UnbinnedDataSet([x]), backend=pf.DeviceBackend())
