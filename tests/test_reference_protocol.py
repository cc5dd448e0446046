"""The drop-in boundary against the REAL reference (the unmodified parafit
installed in baseline/_ref), on CPU.

The reference's own `parafit.engine.nll` (engine.py:214-243) is driven with a
backend whose protocol methods are DeviceBackend's (`block`, `chunk_ranges`,
`map`, engine.py:74-97 / 229-243) and whose device evaluation is replaced by
the oracle -- so this checks, on CPU, exactly the plumbing a reference caller
relies on: the argument layout `map` unpacks, the single `(0, N)` chunk, and
that `math.fsum([total]) == total` hands the device total back unchanged.
"""

import math
import os

import numpy as np
import pytest

from oracle import parafit_oracle as O
from tests import models



class ProtocolBackend:
    """DeviceBackend's reference-facing methods over an oracle evaluation."""

    def __init__(self, spec):
        from paper_1710_08826_b200.engine import DeviceBackend

        self.block = 4096
        self.spec = spec
        self.calls = []
        self.chunk_ranges = DeviceBackend.chunk_ranges.__get__(self)
        self.map = DeviceBackend.map.__get__(self)

    def evaluate(self, pdf, columns, snap, norms, start, stop, index_offset=0):
        self.calls.append((start, stop, index_offset, tuple(sorted(columns))))
        cols = {k: np.asarray(v)[start:stop] for k, v in columns.items()}
        return O.nll(self.spec, cols)


def _reference():
    from paper_1710_08826_b200._reference import core, engine, pdf

    return core, engine, pdf


def test_reference_nll_through_the_backend_protocol():
    core, engine, rpdf = _reference()
    rng = np.random.default_rng(17)
    n = 3 * 4096 + 1234
    x = core.Variable.observable("x", 0.0, 10.0)
    y = core.Variable.observable("y", 0.0, 10.0)
    mu = core.Variable("mu", 5.0, 0.0, 10.0, step=0.01)
    sigma = core.Variable("sigma", 1.0, 0.01, 5.0, step=1e-3)
    alpha = core.Variable("alpha", -0.4, -5.0, 5.0, step=1e-3)
    pdf = rpdf.prod_pdf([rpdf.gaussian(x, mu, sigma), rpdf.exponential(y, alpha)])
    ds = core.UnbinnedDataSet([x, y])
    cx, cy = np.clip(rng.normal(5, 1, n), 0, 10), np.clip(rng.exponential(2.5, n), 0, 10)
    ds.extend([cx, cy])
    backend = ProtocolBackend(models.c2_spec((5.0, 1.0, -0.4)))
    got = engine.nll(pdf, ds, backend=backend)
    # one chunk over the whole range, both observables' columns handed over
    assert backend.calls == [(0, n, 0, ("x", "y"))]
    want = O.nll(models.c2_spec((5.0, 1.0, -0.4)), {"x": cx, "y": cy})
    assert got == want  # fsum([total]) == total: the device value comes back unchanged
    serial = engine.nll(pdf, ds, backend=engine.Backend("serial"))
    assert abs(got - serial) <= 1e-12 * abs(serial)
    assert math.isfinite(got)


def test_backend_rejects_a_foreign_block_size():
    _, engine, _ = _reference()
    backend = ProtocolBackend(models.c2_spec((5.0, 1.0, -0.4)))
    with pytest.raises(ValueError):
        backend.map(lambda *a: None, [(None, {}, None, {}, 0, 10, 1024)])


def test_reference_fitmanager_with_the_backend_protocol(golden_dir):
    """The reference FitManager (fitting.py:410) on the C2 golden events with
    the protocol backend converges to the reference's own fit (fits.json)."""
    import json

    core, engine, rpdf = _reference()
    from parafit.fitting import FitManager

    with open(os.path.join(golden_dir, "fits.json")) as fh:
        ref = json.load(fh)["c2"]
    g = np.load(os.path.join(golden_dir, "c2_prod.npz"))
    x = core.Variable.observable("x", 0.0, 10.0)
    y = core.Variable.observable("y", 0.0, 10.0)
    mu = core.Variable("mu", ref["start"][0], 0.0, 10.0, step=0.01)
    sigma = core.Variable("sigma", ref["start"][1], 0.01, 5.0, step=1e-3)
    alpha = core.Variable("alpha", ref["start"][2], -5.0, 5.0, step=1e-3)
    pdf = rpdf.prod_pdf([rpdf.gaussian(x, mu, sigma), rpdf.exponential(y, alpha)])
    ds = core.UnbinnedDataSet([x, y])
    ds.extend([g["x"], g["y"]])

    class FitBackend(ProtocolBackend):
        def evaluate(self, pdf_, columns, snap, norms, start, stop, index_offset=0):
            spec = models.c2_spec(tuple(snap.value_of(v) for v in (mu, sigma, alpha)))
            cols = {k: np.asarray(v)[start:stop] for k, v in columns.items()}
            return O.nll(spec, cols)

    r = FitManager(pdf, ds, backend=FitBackend(None)).fit()
    assert r.status == "converged" and list(r.names) == ref["names"]
    for v, e, rv, re in zip(r.values, r.errors, ref["values"], ref["errors"]):
        assert abs(v - rv) <= max(1e-6 * abs(rv), 1e-3 * re)
    assert abs(r.nll_min - ref["nll_min"]) <= 1e-10 * abs(ref["nll_min"])
