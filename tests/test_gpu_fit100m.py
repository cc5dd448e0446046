"""North-star target: a 100M-event Dalitz fit converges to the reference's
minimum within tolerance (BASELINE.json north_star).

The events are the reference's own: tests/golden/fit_c4_100m.json was made by
running parafit's generate_dalitz (mcgen.py:157) and FitManager
(fitting.py:410) on 100M events in the builder container
(tests/golden/make_fit100m.py).  Here the device generator redraws the same
100M events from the same GenSpec -- proven by the SHA-256 of both raw
columns -- and the device NLL drives the FitManager from the same start.

Bar: fitted values within 1e-6 relative or 1e-3 sigma, errors within 1e-3
relative, the minimum NLL within 1e-10 relative, the NLL at the start point
within 1e-10 relative.
"""

import hashlib
import json
import math
import os
import time

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

NAMES = ["rhop", "rhom", "rho0", "nr"]


def _host(col) -> np.ndarray:
    if hasattr(col, "detach"):
        col = col.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(col), dtype="<f8")


def run_fit(ref):
    """Generate the reference's 100M events on the device and fit them;
    returns (result, dataset, timings)."""
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200.fitting import DeviceFitManager as FitManager
    from paper_1710_08826_b200.mcgen import GenSpec, generate_dalitz

    start = ref["start"]
    seeded = [(pair, m, w, spin, start.get(f"{nm}_mag", mag), start.get(f"{nm}_ph", ph))
              for nm, (pair, m, w, spin, mag, ph) in zip(NAMES, models.C3_TERMS)]
    (s12, s13), pdf, rts = models.c3(seeded, grid=tuple(ref["grid"]))
    for nm, t in zip(NAMES, rts):
        t.magnitude.name, t.phase.name = f"{nm}_mag", f"{nm}_ph"
    _, _, truth = models.c3(models.C3_TERMS, grid=tuple(ref["grid"]))
    t0 = time.perf_counter()
    gen_stats = {}
    ds = generate_dalitz(truth, P.DecayChannel(*models.D_CHANNEL_T), GenSpec(**ref["spec"]),
                         observables=(s12, s13), stats=gen_stats)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    nll_start = pf.nll(pdf, ds)
    t_first = time.perf_counter() - t0
    t0 = time.perf_counter()
    result = FitManager(pdf, ds).fit()
    t_fit = time.perf_counter() - t0
    return result, ds, {"generate_s": t_gen, "first_nll_s": t_first, "nll_start": nll_start, "fit_s": t_fit,
                        "ambiguous": gen_stats["ambiguous"]}


@pytest.fixture(scope="module")
def ref(golden_dir):
    path = os.path.join(golden_dir, "fit_c4_100m.json")
    with open(path) as fh:
        return json.load(fh)


def test_100m_dalitz_fit_matches_reference(ref):
    result, ds, tm = run_fit(ref)
    assert tm["ambiguous"] == 0  # every accept decision clear of its density by > 2^-47
    cols = ref["columns"]
    for name in ("s12", "s13"):
        a = _host(ds.column(name))
        assert a.shape == (ref["spec"]["n_events"],)
        assert [float(a[i]) for i in cols["rows"]] == cols[name]
        assert hashlib.sha256(a.tobytes()).hexdigest() == cols[f"sha256_{name}"], name
    assert abs(tm["nll_start"] - ref["nll_start"]) <= 1e-10 * abs(ref["nll_start"])
    assert result.status == "converged"
    assert list(result.names) == ref["names"]
    for name, v, e, rv, re in zip(result.names, result.values, result.errors, ref["values"], ref["errors"]):
        tol = max(1e-6 * abs(rv), 1e-3 * re)
        assert abs(v - rv) <= tol, (name, v, rv, tol)
        assert abs(e - re) <= 1e-3 * re, (name, e, re)
    assert abs(result.nll_min - ref["nll_min"]) <= 1e-10 * abs(ref["nll_min"])
    assert math.isfinite(tm["fit_s"])
