"""Persistent evaluation (pfb_objective_set_persistent, nll_persist_kernel):
a kernel resident between minimiser calls, fed through a mapped doorbell.

Every value must be bitwise the one-shot launch's (same canonical blocks),
for C1 (product mode), C2 (unit sums) and C3 (Dalitz ratio form), ragged
sizes included; the exact fix-up (deferred blocks), reference errors, other
device work in between (the resident kernel is stopped and restarted), and
an idle exit (no call for > 20 ms) must all keep the values right.
"""

import math
import time

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


def _fcns(pf, pdf, ds):
    """(persistent, one-shot) C objectives of the same model and data."""
    from paper_1710_08826_b200.fitting import FastObjective

    a = pf.DeviceFitManager(pdf, ds, persistent=True).fcn()
    b = pf.DeviceFitManager(pdf, ds, persistent=False).fcn()
    assert isinstance(a._objective, FastObjective) and isinstance(b._objective, FastObjective)
    return a, b


def _model(cfg, n, seed=5):
    rng = np.random.default_rng(seed)
    if cfg == "c1":
        x, pdf, params = models.c1()
        xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
        return pdf, params, models.dataset([x], [xs])
    if cfg == "c2":
        (x, y), pdf, params = models.c2()
        return pdf, params, models.dataset([x, y], [np.clip(rng.normal(5, 1, n), 0, 10),
                                                    np.clip(rng.exponential(2.5, n), 0, 10)])
    from paper_1710_08826_b200 import mcgen

    terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
    a, b = mcgen.device_dalitz(n, terms, models.D_CHANNEL_T, seed)
    (o12, o13), pdf, rts = models.c3(grid=(96, 96))
    params = [v for t in rts for v in (t.magnitude, t.phase) if not v.fixed]
    return pdf, params, models.dataset([o12, o13], [a, b])


@pytest.mark.parametrize("cfg,n", [("c1", 4096), ("c1", 7 * 4096 + 333), ("c1", 1_000_003), ("c2", 5 * 4096 + 1),
                                   ("c2", 2_000_000), ("c3", 300_001), ("c3", 4097)])
def test_persistent_bitwise_one_shot(pf, cfg, n):
    pdf, params, ds = _model(cfg, n)
    a, b = _fcns(pf, pdf, ds)
    base = np.array([v.value for v in params])
    rng = np.random.default_rng(2)
    for i in range(40):
        pt = base * (1.0 + 0.002 * rng.standard_normal(len(base)))
        assert a(pt) == b(pt), (cfg, n, i)
    a._objective.release()


def test_fixup_errors_and_interleaved_work(pf):
    pdf, params, ds = _model("c1", 200_000)
    params[2].lower = -50.0  # room for |alpha x| beyond the product-mode certification
    a, b = _fcns(pf, pdf, ds)
    base = np.array([v.value for v in params])
    assert a(base) == b(base)
    # |alpha x| beyond the product-mode certification: deferred blocks, exact fix-up
    far = base.copy()
    far[2] = -40.0
    assert a(far) == b(far)
    assert a(base) == b(base)  # the resident kernel restarts
    # interleaved device work on the same context: an ordinary NLL launch
    other = P.nll(pdf, ds, backend=pf.DeviceBackend())
    assert math.isfinite(other)
    assert a(base) == b(base)
    # an error: the same exception as the reference path
    x = P.Variable.observable("x", 0.0, 1.0)
    c0, c1 = P.Variable("c0", 0.5, 0.0, 2.0), P.Variable("c1", 1.0, 0.0, 2.0)
    node = P.prod_pdf([P.gaussian(x, P.Variable("m", 0.5, 0.0, 1.0), P.Variable("s", 0.2, 0.01, 1.0)),
                       P.exponential(P.Variable.observable("y", 0.0, 1.0), P.Variable("al", -0.5, -2.0, 2.0))])
    rng = np.random.default_rng(0)
    dsx = models.dataset(node.observables, [rng.uniform(0, 1, 9000), rng.uniform(0, 1, 9000)])
    ax, bx = _fcns(pf, node, dsx)
    ok = np.array([0.5, 0.2, -0.5])
    assert ax(ok) == bx(ok)
    tiny = np.array([0.0, 0.01, -0.5])  # gaussian underflows to 0 at x ~ 1: NonPositiveDensity
    with pytest.raises(E.NonPositiveDensity) as e1:
        ax(tiny)
    with pytest.raises(E.NonPositiveDensity) as e2:
        bx(tiny)
    assert e1.value.index == e2.value.index
    assert ax(ok) == bx(ok)
    ax._objective.release()
    a._objective.release()


def test_idle_exit_and_restart(pf):
    pdf, params, ds = _model("c2", 100_000)
    a, b = _fcns(pf, pdf, ds)
    base = np.array([v.value for v in params])
    assert a(base) == b(base)
    time.sleep(0.08)  # > 20 ms: the resident kernel leaves by itself
    for k in range(3):
        pt = base * (1.0 + 1e-3 * k)
        assert a(pt) == b(pt)
    a._objective.release()


def test_persistent_fit_bitwise_and_gpu_released(pf):
    pdf, params, ds = _model("c1", 500_000)
    start = (4.8, 0.6, -0.25, 0.35)
    res = []
    for persistent in (True, False):
        for v, val in zip(params, start):
            P.set_value(v, val)
        fm = pf.DeviceFitManager(pdf, ds, persistent=persistent)
        res.append(fm.fit())
    assert res[0].n_calls == res[1].n_calls
    assert np.array_equal(res[0].values, res[1].values) and res[0].nll_min == res[1].nll_min
    import torch

    torch.cuda.synchronize()  # the fit stopped its resident kernel: a device-wide sync returns
