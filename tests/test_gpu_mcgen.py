"""Device toy generation (pfb_gen_1d / pfb_gen_dalitz): determinism per seed,
support, and agreement with the model (moments, and the fitted truth)."""

import math

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mc():
    from paper_1710_08826_b200 import _lib as L
    from paper_1710_08826_b200 import mcgen

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return mcgen


def test_prod_2d_deterministic_and_moments(mc):
    x1, y1 = mc.device_prod_2d(400_000, 5.0, 1.0, -0.4, 0.0, 10.0, seed=7)
    x2, y2 = mc.device_prod_2d(400_000, 5.0, 1.0, -0.4, 0.0, 10.0, seed=7)
    x3, _ = mc.device_prod_2d(400_000, 5.0, 1.0, -0.4, 0.0, 10.0, seed=8)
    assert np.array_equal(x1, x2) and np.array_equal(y1, y2)
    assert not np.array_equal(x1, x3)
    assert x1.min() >= 0.0 and x1.max() <= 10.0 and y1.min() >= 0.0 and y1.max() <= 10.0
    assert abs(x1.mean() - 5.0) < 5 * 1.0 / math.sqrt(len(x1))
    assert abs(x1.std() - 1.0) < 0.01
    # truncated exponential mean on [0, 10] with alpha = -0.4
    a = -0.4
    mean = (10 * math.exp(10 * a) / (math.exp(10 * a) - 1)) - 1 / a
    assert abs(y1.mean() - mean) < 0.01


def test_sumpdf_fraction(mc):
    x = mc.device_sumpdf_1d(500_000, 5.0, 0.2, -0.3, 0.3, 0.0, 10.0, seed=3)
    near = np.mean(np.abs(x - 5.0) < 1.0)  # gaussian mass within 5 sigma + exponential share
    a = -0.3
    norm = (math.exp(10 * a) - 1) / a
    exp_share = (math.exp(6 * a) - math.exp(4 * a)) / a / norm
    assert abs(near - (0.3 + 0.7 * exp_share)) < 0.005


def test_dalitz_generation_inside_and_fit_truth(mc):
    import paper_1710_08826_b200 as pf

    terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in models.C3_TERMS]
    s12, s13 = mc.device_dalitz(300_000, terms, models.D_CHANNEL_T, seed=11)
    s12b, _ = mc.device_dalitz(300_000, terms, models.D_CHANNEL_T, seed=11)
    assert np.array_equal(s12, s12b)
    ch = P.DecayChannel(*models.D_CHANNEL_T)
    from paper_1710_08826_b200._reference import dalitz as RD

    in_boundary_mask = RD.in_boundary_mask

    assert in_boundary_mask(s12, s13, ch).all()
    # the generating coefficients give a lower NLL than perturbed ones
    (o12, o13), pdf, rts = models.c3()
    ds = models.dataset([o12, o13], [s12, s13])
    truth = pf.nll(pdf, ds)
    P.set_value(rts[1].magnitude, 0.9)
    assert pf.nll(pdf, ds) > truth + 10.0
