"""Device normalisation integrals behind the reference's norm cache
(north_star item 4).

* The reference's cache tests (T/test_engine.py:125-185,
  T/test_dalitz.py:372-386,410-463) re-run with the device hooks installed:
  zero kernel evaluations on a repeat, fraction-only recomputes, a child
  change re-integrates only that child, warm == cold bitwise over random
  interleavings, Dalitz coefficient moves reuse the matrix, a floating-mass
  fit recomputes only the floating term's rows.
* The device Gauss-Legendre quadrature against the reference's own
  ``_polynomial_norm`` (P/pdf.py:192-199, <= 1e-12) and closed forms
  (P/pdf.py:130-161, <= 1e-10), in 1-D and on the 2-D tensor grid of the C2
  product; error semantics as the reference (index into the abscissa array).
"""

import math

import numpy as np
import pytest

from paper_1710_08826_b200._reference import parafit as P
from paper_1710_08826_b200._reference import pdf as ref_pdf
from tests import models

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    pf.device_context(0)
    return pf


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# --- the reference's cache tests on the device hooks ------------------------------------


def poly_tree():
    """add(polynomial, polynomial): both leaves integrate on the device."""
    x = P.Variable.observable("x", 0.0, 1.0)
    p1 = P.polynomial(x, [P.Variable("a0", 1.0, 0.1, 3.0), P.Variable("a1", 0.4, -0.5, 0.5)])
    p2 = P.polynomial(x, [P.Variable("b0", 0.5, 0.1, 3.0), P.Variable("b1", 0.2, -0.1, 0.3),
                          P.Variable("b2", 0.3, 0.0, 1.0)])
    frac = P.Variable("f", 0.4, 0.0, 1.0)
    return x, P.add_pdf([p1, p2], [frac]), (p1, p2, frac)


def test_repeat_call_zero_kernel_evals(pf):
    x, tree, _ = poly_tree()
    store = P.NormalizationStore()
    snap = P.snapshot(tree.param_closure())
    P.resolve_norms(tree, snap, store)
    assert store.kernel_evals == 2  # two leaf integrals, on the device
    before = store.kernel_evals
    P.resolve_norms(tree, snap, store)
    assert store.kernel_evals == before


def test_fraction_change_recomputes_only_add_node(pf):
    x, tree, (p1, p2, frac) = poly_tree()
    store = P.NormalizationStore()
    P.resolve_norms(tree, P.snapshot(tree.param_closure()), store)
    kernel_before = store.kernel_evals
    counts_before = dict(store.recompute_counts)
    P.set_value(frac, 0.5)
    P.resolve_norms(tree, P.snapshot(tree.param_closure()), store)
    assert store.kernel_evals == kernel_before
    assert store.recompute_counts[tree.id] == counts_before[tree.id] + 1
    assert store.recompute_counts[p1.id] == counts_before[p1.id]
    assert store.recompute_counts[p2.id] == counts_before[p2.id]


def test_child_change_recomputes_child_and_parent(pf):
    x, tree, (p1, p2, frac) = poly_tree()
    store = P.NormalizationStore()
    P.resolve_norms(tree, P.snapshot(tree.param_closure()), store)
    kernel_before = store.kernel_evals
    P.set_value(p1.parameters[1], 0.35)
    P.resolve_norms(tree, P.snapshot(tree.param_closure()), store)
    assert store.kernel_evals == kernel_before + 1  # only p1 re-integrated (on the device)


def test_randomized_interleavings_warm_equals_cold(pf):
    rng = np.random.default_rng(7)
    x, tree, (p1, p2, frac) = poly_tree()
    params = [p1.parameters[0], p1.parameters[1], p2.parameters[0], p2.parameters[2], frac]
    store = P.NormalizationStore()
    for _ in range(300):
        var = params[rng.integers(len(params))]
        set_to = float(rng.uniform(max(var.lower, 0.02), min(var.upper, 0.98)))
        P.set_value(var, set_to)
        snap = P.snapshot(tree.param_closure())
        warm = P.resolve_norms(tree, snap, store)
        cold = P.resolve_norms(tree, snap, P.NormalizationStore())
        assert warm == cold


def test_device_polynomial_norm_matches_reference(pf):
    x, tree, (p1, p2, frac) = poly_tree()
    for node in (p1, p2):
        dev = P.cached_norm(node, None, P.NormalizationStore()).value
        with pf.reference_norms():
            want = P.cached_norm(node, None, P.NormalizationStore()).value
        assert rel(dev, want) <= 1e-12, (dev, want)
        assert rel(dev, ref_pdf._polynomial_norm(node, None, {})) <= 1e-12


def test_grid_mode_gaussian_tree_counters_and_closed_forms(pf):
    """The reference's own TestNormCache tree (two gaussians) with the opt-in
    device grid norms: same counters as the closed forms, values <= 1e-10."""
    x = P.Variable.observable("x", 0.0, 1.0)
    g1 = P.gaussian(x, P.Variable("mu1", 0.3, 0.0, 1.0), P.Variable("s1", 0.1, 1e-3, 1.0))
    g2 = P.gaussian(x, P.Variable("mu2", 0.7, 0.0, 1.0), P.Variable("s2", 0.08, 1e-3, 1.0))
    tree = P.add_pdf([g1, g2], [P.Variable("f", 0.4, 0.0, 1.0)])
    with pf.reference_norms():
        s_ref = P.NormalizationStore()
        want = P.resolve_norms(tree, P.snapshot(tree.param_closure()), s_ref)
    with pf.device_norms(grid_kinds=("gaussian",)):
        s_dev = P.NormalizationStore()
        got = P.resolve_norms(tree, P.snapshot(tree.param_closure()), s_dev)
        P.resolve_norms(tree, P.snapshot(tree.param_closure()), s_dev)
        P.set_value(g1.parameters[0], 0.35)
        P.resolve_norms(tree, P.snapshot(tree.param_closure()), s_dev)
    assert s_dev.kernel_evals == 3  # two leaves, then g1 again
    for k in want:
        assert rel(got[k], want[k]) <= 1e-10
    assert ref_engine_hook("gaussian") is None  # grid mode left again


def ref_engine_hook(kind):
    from paper_1710_08826_b200._reference import engine

    return engine.CACHED_NORM_HOOKS.get(kind)


# --- quadrature against the closed forms (J1) ----------------------------------------------


def test_quadrature_1d_closed_forms(pf):
    x = P.Variable.observable("x", 0.0, 10.0)
    cases = [P.gaussian(x, P.Variable("m", 5.0), P.Variable("s", 1.0)),
             P.gaussian(x, P.Variable("m2", 3.3, fixed=True), P.Variable("s2", 0.7, fixed=True)),
             P.exponential(x, P.Variable("a", -0.4)),
             P.exponential(x, P.Variable("a2", 0.25))]
    for node in cases:
        got = pf.quadrature(node)
        want = ref_pdf.KIND_OPS[node.kind][1](node, None, {})
        assert rel(got, want) <= 1e-10, (node.kind, got, want)


def test_quadrature_2d_grid_of_the_c2_product(pf):
    """C2's product over the 2-D tensor GL grid (1024 x 1024 nodes): with unit
    child norms it integrates to the product of the closed-form norms; with the
    children's own norms, to 1."""
    (x, y), pdf, (mu, sigma, alpha) = models.c2()
    g, e = pdf.children
    ng = ref_pdf._gaussian_norm(g, None, {})
    ne = ref_pdf._exponential_norm(e, None, {})
    raw = pf.quadrature(pdf, child_norms={g.id: 1.0, e.id: 1.0})
    assert rel(raw, ng * ne) <= 1e-10, (raw, ng * ne)
    unit = pf.quadrature(pdf, child_norms={g.id: ng, e.id: ne})
    assert abs(unit - 1.0) <= 1e-10
    P.set_value(sigma, 0.6)
    P.set_value(alpha, -0.9)
    raw = pf.quadrature(pdf, child_norms={g.id: 1.0, e.id: 1.0})
    want = ref_pdf._gaussian_norm(g, None, {}) * ref_pdf._exponential_norm(e, None, {})
    assert rel(raw, want) <= 1e-10


def test_quadrature_errors_as_reference(pf):
    from paper_1710_08826_b200._reference import errors as E

    x = P.Variable.observable("x", 0.0, 1.0)
    dip = P.polynomial(x, [0.01, -1.0, 1.0])  # negative around x = 0.5
    with pytest.raises(E.NegativeDensity) as ref_err:
        ref_pdf._polynomial_norm(dip, None, {})
    with pytest.raises(E.NegativeDensity) as dev_err:
        P.cached_norm(dip, None, P.NormalizationStore())
    assert dev_err.value.index == ref_err.value.index
    assert dev_err.value.value == ref_err.value.value
    u = P.Variable.observable("u", 0.0, math.inf)
    with pytest.raises(E.UnboundedObservable):
        P.cached_norm(P.polynomial(u, [1.0, 0.5]), None, P.NormalizationStore())


def test_nll_with_device_polynomial_norm_matches_reference(pf):
    """C2 with a polynomial factor (the variant on the bench's timed path): the
    device GL norm inside the reference nll, vs the reference end to end."""
    rng = np.random.default_rng(5)
    n = 300_017
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    c = [P.Variable("c0", 1.0, 0.1, 5.0), P.Variable("c1", 0.3, -0.05, 1.0), P.Variable("c2", 0.05, 0.0, 1.0)]
    pdf = P.prod_pdf([P.gaussian(x, P.Variable("mu", 5.0, 0.0, 10.0), P.Variable("sg", 1.0, 0.1, 5.0)),
                      P.polynomial(y, c)])
    ds = models.dataset([x, y], [np.clip(rng.normal(5, 1, n), 0, 10), rng.uniform(0, 10, n)])
    store = P.NormalizationStore()
    for c1 in (0.3, 0.31, 0.29):
        P.set_value(c[1], c1)
        got = P.nll(pdf, ds, None, pf.DeviceBackend(), store)
        with pf.reference_norms():
            want = P.nll(pdf, ds, None, P.Backend("serial"))
        assert rel(got, want) <= 1e-10
    assert store.kernel_evals == 1 + 3  # gaussian closed form once, polynomial per move


# --- Dalitz (T/test_dalitz.py:372-386, 410-463) -------------------------------------------


def _term(pair, name, mass=0.77526, width=0.1478, spin=1, mag=1.0, phase=0.0):
    return P.ResonanceTerm(pair, P.Variable(f"{name}_m", mass, fixed=True), P.Variable(f"{name}_w", width, fixed=True),
                           spin, P.Variable(f"{name}_c", mag, fixed=True), P.Variable(f"{name}_p", phase, fixed=True))


def test_dalitz_coefficient_change_reuses_matrix(pf):
    ch = P.DecayChannel(*models.D_CHANNEL_T)
    mag = P.Variable("mag_free", 1.0, 0.0, 10.0, step=0.01)
    terms = [_term(12, "fixed"),
             P.ResonanceTerm(13, P.Variable("mm", 0.9, fixed=True), P.Variable("ww", 0.05, fixed=True), 0, mag,
                             P.Variable("pp", 0.3, fixed=True))]
    node = P.dalitz_pdf(terms, ch, grid=(48, 48))
    store = P.NormalizationStore()
    P.resolve_norms(node, P.snapshot(node.param_closure()), store)
    assert store.kernel_evals == 2
    P.set_value(mag, 2.0)
    norms = P.resolve_norms(node, P.snapshot(node.param_closure()), store)
    assert store.kernel_evals == 2
    with pf.reference_norms():
        want = P.resolve_norms(node, P.snapshot(node.param_closure()), P.NormalizationStore())
    assert rel(norms[node.id], want[node.id]) <= 1e-12


def test_dalitz_warm_equals_cold_with_floating_shape(pf):
    rng = np.random.default_rng(13)
    ch = P.DecayChannel(*models.D_CHANNEL_T)
    mass = P.Variable("wc_m", 0.9, 0.7, 1.1, step=0.001)
    mag = P.Variable("wc_c", 1.0, 0.0, 5.0, step=0.01)
    terms = [_term(12, "wca"),
             P.ResonanceTerm(13, mass, P.Variable("wc_w", 0.05, fixed=True), 0, mag,
                             P.Variable("wc_p", 0.2, fixed=True))]
    node = P.dalitz_pdf(terms, ch, grid=(48, 48))
    store = P.NormalizationStore()
    for _ in range(60):
        var = mass if rng.random() < 0.5 else mag
        P.set_value(var, float(rng.uniform(var.lower + 0.01, var.upper - 0.01)))
        snap = P.snapshot(node.param_closure())
        warm = P.resolve_norms(node, snap, store)[node.id]
        cold = P.resolve_norms(node, snap, P.NormalizationStore())[node.id]
        assert warm == cold


def test_dalitz_fit_with_floating_mass_reuses_fixed_rows(pf):
    """The reference's floating-mass fit on the device: only the floating
    term's row is recomputed per shape move, and the truth is recovered."""
    from paper_1710_08826_b200 import mcgen

    ch = P.DecayChannel(*models.D_CHANNEL_T)
    truth = [_term(12, "ta"), _term(13, "tb", mass=0.892, width=0.051, mag=1.4, phase=0.8, spin=0)]
    ds = mcgen.generate_dalitz(truth, ch, P.GenSpec(n_events=20_000, seed=41))
    mass_b = P.Variable("fit_mb", 0.90, 0.80, 1.00, step=0.001)
    mag_b = P.Variable("fit_cb", 1.0, 0.0, 10.0, step=0.01)
    model = [_term(12, "fa"),
             P.ResonanceTerm(13, mass_b, P.Variable("fit_wb", 0.051, fixed=True), 0, mag_b,
                             P.Variable("fit_pb", 0.8, fixed=True))]
    node = P.dalitz_pdf(model, ch, s12_obs=ds.observables[0], s13_obs=ds.observables[1], grid=(96, 96))
    manager = pf.DeviceFitManager(node, ds)
    result = manager.fit()
    assert result.status == "converged"
    by = dict(zip(result.names, result.values))
    errs = dict(zip(result.names, result.errors))
    assert abs(by["fit_mb"] - 0.892) <= 4 * errs["fit_mb"]
    assert abs(by["fit_cb"] - 1.4) <= 4 * errs["fit_cb"]
    # the fixed term integrates once, the floating term once per mass move
    # (coefficient-only moves recompute the node's norm, not its rows)
    evals = manager.store.kernel_evals
    recomputes = manager.store.recompute_counts[node.id]
    assert evals >= 3 and recomputes >= 3
    assert evals <= 1 + recomputes
