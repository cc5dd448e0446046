"""Stream-exact toy generation: the device generators
reproduce the reference's generate_1d / generate_dalitz events, statistics,
envelope rescans and errors for the same GenSpec (fixtures: the real
reference, tests/golden/make_golden.py toys_fixture)."""

import os

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


@pytest.fixture(scope="module")
def g(golden_dir):
    return np.load(os.path.join(golden_dir, "toys.npz"))


def check_stats(stats, want, keys):
    assert abs(stats["envelope"] - want[0]) <= 1e-15 * abs(want[0])
    # no accept decision within 2^-47 of its density: the run is exact by
    # construction, not only equal to the fixture
    assert stats["ambiguous"] == 0
    for k, w in zip(keys, want[1:]):
        assert stats[k] == int(w), k


@pytest.mark.parametrize("tag,spec", [("a", dict(n_events=20000, seed=5)),
                                      ("b", dict(n_events=10001, seed=9, streams=3))])
def test_generate_1d_equals_reference(pf, g, tag, spec):
    from paper_1710_08826_b200.mcgen import GenSpec, generate_1d  # GenSpec: the reference's

    x, pdf, _ = models.c1()
    stats = {}
    ds = generate_1d(pdf, x, GenSpec(**spec), stats)
    assert ds.column("x").tolist() == g[f"c1{tag}_x"].tolist()
    check_stats(stats, g[f"c1{tag}_stats"], ("attempts", "accepted"))


def test_envelope_rescan_exceeded_and_budget(pf, g):
    from paper_1710_08826_b200._reference import errors as E
    from paper_1710_08826_b200.mcgen import GenSpec, generate_1d  # GenSpec: the reference's

    xs = P.Variable.observable("x", 0.0, 10.0)
    spike = P.gaussian(xs, P.Variable("m", 5.00061, 0.0, 10.0), P.Variable("s", 0.001, 1e-5, 1.0))
    stats = {}
    ds = generate_1d(spike, xs, GenSpec(300, seed=2, max_attempts_factor=100000), stats)
    assert ds.column("x").tolist() == g["spike_x"].tolist()
    check_stats(stats, g["spike_stats"], ("attempts", "accepted"))
    narrow = P.gaussian(xs, P.Variable("m2", 5.00061, 0.0, 10.0), P.Variable("s2", 0.0005, 1e-5, 1.0))
    assert int(g["narrow_exceeded"][0]) == 1
    with pytest.raises(E.EnvelopeExceeded):
        generate_1d(narrow, xs, GenSpec(300, seed=2, max_attempts_factor=100000))
    with pytest.raises(E.AttemptsExhausted) as ei:
        generate_1d(spike, xs, GenSpec(300, seed=2))
    assert str(ei.value) == str(g["spike_exhausted"][0])


@pytest.mark.parametrize("tag,spec", [("a", dict(n_events=3000, seed=3)),
                                      ("b", dict(n_events=2001, seed=4, streams=2))])
def test_generate_dalitz_equals_reference(pf, g, tag, spec):
    from paper_1710_08826_b200.mcgen import GenSpec, generate_dalitz

    _, _, terms = models.c3()
    stats = {}
    ds = generate_dalitz(terms, P.DecayChannel(*models.D_CHANNEL_T), GenSpec(**spec), stats=stats)
    assert ds.column("s12").tolist() == g[f"dal{tag}_s12"].tolist()
    assert ds.column("s13").tolist() == g[f"dal{tag}_s13"].tolist()
    check_stats(stats, g[f"dal{tag}_stats"], ("box_draws", "in_boundary_draws", "accepted"))
