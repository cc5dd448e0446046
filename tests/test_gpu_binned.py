"""Binned data on the device against the reference's golden
outputs: BinnedDataSet.fill bit-exact, binned_nll within 1e-10, the reference's
errors, and a binned fit through FitManager."""

import os

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

RTOL = 1e-10


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


@pytest.fixture(scope="module")
def g(golden_dir):
    return np.load(os.path.join(golden_dir, "binned.npz"))


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def test_fill_bitwise_1d(pf, g):
    x, pdf, params = models.c1()
    ds = models.dataset([x], [g["b1_x"]])
    b = P.BinnedDataSet([x], [100])
    pf.bin_fill(b, ds)
    assert b.contents.tolist() == g["b1_contents"].tolist()
    pf.bin_fill(b, ds)  # fill accumulates like np.add.at
    assert b.contents.tolist() == (2 * g["b1_contents"]).tolist()


def test_fill_bitwise_2d_and_nll(pf, g):
    (x, y), pdf, params = models.c2()
    ds = models.dataset([x, y], [g["b2_x"], g["b2_y"]])
    b = P.BinnedDataSet([x, y], [40, 25])
    pf.bin_fill(b, ds)
    assert b.contents.tolist() == g["b2_contents"].tolist()
    for pt, want in zip(g["b2_points"], g["b2_nll"]):
        for v, val in zip(params, pt):
            P.set_value(v, float(val))
        assert rel(pf.binned_nll(pdf, b), want) <= RTOL


def test_binned_nll_1d(pf, g):
    x, pdf, params = models.c1()
    b = P.BinnedDataSet([x], [100])
    b.contents[:] = g["b1_contents"]
    for pt, want in zip(g["b1_points"], g["b1_nll"]):
        for v, val in zip(params, pt):
            P.set_value(v, float(val))
        assert rel(pf.binned_nll(pdf, b), want) <= RTOL


def test_nonpositive_expectation_and_empty(pf, g):
    from paper_1710_08826_b200._reference import errors as E

    x = P.Variable.observable("x", 0.0, 1.0)
    pdf = P.gaussian(x, P.Variable("gm", 0.5, 0.0, 1.0), P.Variable("gs", 0.01, 0.001, 1.0))
    b = P.BinnedDataSet([x], [20])
    with pytest.raises(E.EmptyDataSet):
        pf.binned_nll(pdf, b)
    b.contents[:] = g["bp_contents"]
    with pytest.raises(E.NonPositiveExpectation) as ei:
        pf.binned_nll(pdf, b)
    assert ei.value.bin_index == int(g["bp_bin"][0]) and ei.value.value == float(g["bp_value"][0])


def test_binned_fit_matches_reference(pf, g):
    from paper_1710_08826_b200.fitting import DeviceFitManager as FitManager

    (x, y), pdf, params = models.c2((4.9, 1.1, -0.35))
    b = P.BinnedDataSet([x, y], [40, 25])
    b.contents[:] = g["b2_contents"]
    r = FitManager(pdf, b).fit()
    want, err = g["b2_fit_values"], g["b2_fit_errors"]
    for v, w, e in zip(r.values, want, err):
        assert abs(v - w) <= max(1e-6 * abs(w), 1e-3 * e)
    assert rel(r.nll_min, float(g["b2_fit_nll"][0])) <= RTOL
