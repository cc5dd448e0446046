"""Fit parity: the device NLL driving the fitter reproduces the reference
FitManager's minimum (tests/golden/fits.json, produced by the real parafit).

Bar (north_star): fitted parameters within 1e-6 relative or 1e-3 sigma; the
minimum NLL within 1e-10 relative.
"""

import json
import math
import os

import numpy as np
import pytest

from tests import models

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fits(golden_dir):
    with open(os.path.join(golden_dir, "fits.json")) as fh:
        return json.load(fh)


def check(result, ref):
    assert result.status == "converged"
    assert list(result.names) == ref["names"]
    for name, v, e, rv, re in zip(result.names, result.values, result.errors, ref["values"], ref["errors"]):
        tol = max(1e-6 * abs(rv), 1e-3 * re)
        assert abs(v - rv) <= tol, (name, v, rv, tol)
        assert abs(e - re) <= 1e-3 * re, (name, e, re)
    assert abs(result.nll_min - ref["nll_min"]) <= 1e-10 * abs(ref["nll_min"])


def test_c1_fit_matches_reference(fits, golden_dir):
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200.fitting import DeviceFitManager as FitManager

    g = np.load(os.path.join(golden_dir, "c1_sumpdf.npz"))
    x, pdf, params = models.c1(tuple(fits["c1"]["start"]))
    ds = models.dataset([x], [g["x"]])
    check(FitManager(pdf, ds).fit(), fits["c1"])


def test_c2_fit_matches_reference(fits, golden_dir):
    from paper_1710_08826_b200.fitting import DeviceFitManager as FitManager

    g = np.load(os.path.join(golden_dir, "c2_prod.npz"))
    (x, y), pdf, params = models.c2(tuple(fits["c2"]["start"]))
    ds = models.dataset([x, y], [g["x"], g["y"]])
    check(FitManager(pdf, ds).fit(), fits["c2"])


def test_c3_dalitz_fit_matches_reference(fits, golden_dir):
    from paper_1710_08826_b200.fitting import DeviceFitManager as FitManager

    g = np.load(os.path.join(golden_dir, "c3_dalitz.npz"))
    ref = fits["c3"]
    start = ref["start"]
    terms = list(models.C3_TERMS)
    names = ["rhop", "rhom", "rho0", "nr"]
    seeded = []
    for nm, (pair, m, w, spin, mag, ph) in zip(names, terms):
        seeded.append((pair, m, w, spin, start.get(f"{nm}_mag", mag), start.get(f"{nm}_ph", ph)))
    (s12, s13), pdf, rts = models.c3(seeded, grid=tuple(ref["grid"]))
    for nm, t in zip(names, rts):
        t.magnitude.name, t.phase.name = f"{nm}_mag", f"{nm}_ph"
    ds = models.dataset([s12, s13], [g["s12"], g["s13"]])
    check(FitManager(pdf, ds).fit(), ref)
