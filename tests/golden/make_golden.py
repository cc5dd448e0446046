"""Generate golden fixtures by running the REAL reference (parafit) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is imported from /root/reference/pkg/src (read-only, never
copied).  Inputs are drawn with fixed numpy seeds and stored next to the
reference outputs, so the GPU box -- which has no /root/reference -- checks
the device engine against exactly these numbers.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
os.environ.pop("PARAFIT_WORKERS", None)

from parafit.core import UnbinnedDataSet, Variable, snapshot  # noqa: E402
from parafit.dalitz import (  # noqa: E402
    DecayChannel,
    ResonanceTerm,
    compute_integrals,
    dalitz_norm,
    dalitz_pdf,
    integration_grid,
)
from parafit.engine import Backend, NormalizationStore, nll, nll_block_sums, resolve_norms  # noqa: E402
from parafit.errors import ParafitError  # noqa: E402
from parafit.mcgen import GenSpec, generate_dalitz  # noqa: E402
from parafit.pdf import add_pdf, exponential, gaussian, polynomial, prod_pdf  # noqa: E402
from parafit.reduction import block_sums  # noqa: E402
from parafit.sharding import shard, sharded_nll  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
D_CHANNEL = DecayChannel(1.86484, 0.13957, 0.13957, 0.13498)


def reduction_fixture():
    rng = np.random.default_rng(101)
    sizes = [1, 7, 8, 9, 13, 100, 257, 1000, 4095, 4096, 4097, 8191, 3 * 4096 + 1234]
    out = {}
    for n in sizes:
        terms = rng.normal(size=n) * 10.0 ** rng.integers(-6, 7, size=n)
        bs = block_sums(terms, 4096)
        out[f"terms_{n}"] = terms
        out[f"bsums_{n}"] = bs
        out[f"total_{n}"] = np.array([math.fsum(bs.tolist())])
    # cancellation-heavy case: a large multiple of the block, exact-sum sensitive
    terms = np.concatenate([rng.normal(size=20480) * 1e16, rng.normal(size=20480)])
    rng.shuffle(terms)
    bs = block_sums(terms, 4096)
    out["terms_cancel"] = terms
    out["bsums_cancel"] = bs
    out["total_cancel"] = np.array([math.fsum(bs.tolist())])
    np.savez_compressed(os.path.join(OUT, "reduction.npz"), **out)


def c1_model():
    x = Variable.observable("x", 0.0, 10.0)
    mu = Variable("mu", 5.0, 0.0, 10.0, step=0.01)
    sigma = Variable("sigma", 0.5, 0.01, 5.0, step=1e-3)
    alpha = Variable("alpha", -0.3, -5.0, 5.0, step=1e-3)
    f = Variable("f", 0.3, 0.0, 1.0, step=1e-3)
    return x, add_pdf([gaussian(x, mu, sigma), exponential(x, alpha)], [f]), (mu, sigma, alpha, f)


def c1_fixture():
    rng = np.random.default_rng(7)
    n = 3 * 4096 + 1500
    xs = np.concatenate([np.clip(rng.normal(5.0, 0.5, n // 3), 0, 10), rng.exponential(1 / 0.3, n - n // 3)])
    xs = xs[(xs >= 0) & (xs <= 10)][: n - 300]
    rng.shuffle(xs)
    x, pdf, params = c1_model()
    ds = UnbinnedDataSet([x])
    ds.extend([xs])
    points = [(5.0, 0.5, -0.3, 0.3), (4.8, 0.6, -0.25, 0.35), (5.3, 0.05, -1.0, 0.999), (5.0, 0.5, 0.7, 0.0)]
    vals, bsums = [], []
    for pt in points:
        for v, value in zip(params, pt):
            v.value = value
        snap = snapshot(pdf.param_closure())
        vals.append(nll(pdf, ds, snap, Backend("serial")))
        assert nll(pdf, ds, snap, Backend("pool", workers=3)) == vals[-1]
        norms = resolve_norms(pdf, snap, NormalizationStore())
        bsums.append(nll_block_sums(pdf, ds.columns(), snap, norms, 0, ds.n_events, 4096))
    np.savez_compressed(os.path.join(OUT, "c1_sumpdf.npz"), x=xs, points=np.array(points), nll=np.array(vals),
                        **{f"bsums_{i}": b for i, b in enumerate(bsums)})


def c2_fixture():
    rng = np.random.default_rng(11)
    n = 5 * 4096 + 77
    xs = np.clip(rng.normal(5.0, 1.0, n), 0, 10)
    ys = np.clip(rng.exponential(1 / 0.4, n), 0, 10)
    x = Variable.observable("x", 0.0, 10.0)
    y = Variable.observable("y", 0.0, 10.0)
    mu = Variable("mu", 5.0, 0.0, 10.0, step=0.01)
    sigma = Variable("sigma", 1.0, 0.01, 5.0, step=1e-3)
    alpha = Variable("alpha", -0.4, -5.0, 5.0, step=1e-3)
    pdf = prod_pdf([gaussian(x, mu, sigma), exponential(y, alpha)])
    ds = UnbinnedDataSet([x, y])
    ds.extend([xs, ys])
    points = [(5.0, 1.0, -0.4), (4.9, 1.1, -0.35), (2.0, 0.3, 0.5)]
    vals = []
    for pt in points:
        mu.value, sigma.value, alpha.value = pt
        vals.append(nll(pdf, ds, snapshot(pdf.param_closure()), Backend("serial")))
    sh = {}
    for w in (2, 3, 4):
        mu.value, sigma.value, alpha.value = points[0]
        sh[f"sharded_{w}"] = np.array([sharded_nll(pdf, ds, snapshot(pdf.param_closure()), workers=w)])
    np.savez_compressed(os.path.join(OUT, "c2_prod.npz"), x=xs, y=ys, points=np.array(points), nll=np.array(vals),
                        **sh)


def c3_terms():
    def term(pair, m, w, spin, mag, ph, name, fix_coef=False):
        return ResonanceTerm(
            pair=pair,
            mass=Variable(f"{name}_m", m, fixed=True),
            width=Variable(f"{name}_w", w, fixed=True),
            spin=spin,
            magnitude=Variable(f"{name}_mag", mag, 0.0, 100.0, step=0.01, fixed=fix_coef),
            phase=Variable(f"{name}_ph", ph, -2 * math.pi, 2 * math.pi, step=0.01, fixed=fix_coef),
            name=name,
        )

    return [
        term(13, 0.77511, 0.1491, 1, 1.0, 0.0, "rhop", fix_coef=True),
        term(23, 0.77511, 0.1491, 1, 0.73, -0.03, "rhom"),
        term(12, 0.77526, 0.1478, 1, 0.55, 0.28, "rho0"),
        term(12, 1.0, 20.0, 0, 20.0, -0.5, "nr"),
    ]


def c3_fixture():
    terms = c3_terms()
    ds = generate_dalitz(terms, D_CHANNEL, GenSpec(n_events=3 * 4096 + 999, seed=3))
    out = {"s12": ds.column("s12"), "s13": ds.column("s13")}
    # masks and overlap matrices at two grid sizes
    for grid in ((64, 64), (400, 400)):
        g12, g13, mask, darea = integration_grid(D_CHANNEL, grid)
        tag = f"{grid[0]}x{grid[1]}"
        out[f"mask_{tag}"] = np.packbits(mask)
        out[f"ninside_{tag}"] = np.array([int(mask.sum())])
        out[f"darea_{tag}"] = np.array([darea])
        cache = compute_integrals(terms, D_CHANNEL, grid)
        out[f"matrix_{tag}"] = cache.matrix
        out[f"norm_{tag}"] = np.array([dalitz_norm(terms, cache)])
    pdf = dalitz_pdf(terms, D_CHANNEL, s12_obs=ds.observables[0], s13_obs=ds.observables[1], grid=(400, 400))
    snap = snapshot(pdf.param_closure())
    out["nll"] = np.array([nll(pdf, ds, snap, Backend("serial"))])
    norms = resolve_norms(pdf, snap, NormalizationStore())
    out["bsums"] = nll_block_sums(pdf, ds.columns(), snap, norms, 0, ds.n_events, 4096)
    # a second coefficient point
    terms[1].magnitude.value = 0.9
    terms[2].phase.value = 1.1
    out["nll_b"] = np.array([nll(pdf, ds, snapshot(pdf.param_closure()), Backend("serial"))])
    np.savez_compressed(os.path.join(OUT, "c3_dalitz.npz"), **out)


def shards_fixture():
    table = {}
    for n in (0, 1, 7, 10, 100, 1000, 4096, 10_001, 16_384, 10_000_000, 100_000_000):
        for w in (1, 2, 3, 4, 5, 8):
            x = Variable.observable("x")
            ds = UnbinnedDataSet([x])
            if n <= 20000:
                ds.extend([np.zeros(n)])
                b = [s.begin for s in shard(ds, w)] + [n]
            else:  # reference shard() on a stand-in dataset of the same length
                class _DS:
                    n_events = n
                    observables = (x,)

                    def columns(self):
                        return {"x": np.empty(0)}

                b = [s.begin for s in shard(_DS(), w)] + [n]
            table[f"{n}/{w}"] = b
    with open(os.path.join(OUT, "shard_bounds.json"), "w") as fh:
        json.dump(table, fh, indent=0, sort_keys=True)


def errors_fixture():
    cases = {}
    x = Variable.observable("x", 0.0, 1.0)
    node = polynomial(x, [0.0, 1.0])
    values = np.full(5000, 0.5)
    values[4321] = 0.0
    ds = UnbinnedDataSet([x])
    ds.extend([values])
    try:
        nll(node, ds)
    except ParafitError as e:
        cases["poly_zero"] = [type(e).__name__, e.index, e.value]
    node2 = polynomial(x, [0.1, -1.0])  # negative above x = 0.1
    values2 = np.full(9000, 0.05)
    values2[7777] = 0.5
    values2[8000] = 0.9
    ds2 = UnbinnedDataSet([x])
    ds2.extend([values2])
    try:
        nll(node2, ds2)
    except ParafitError as e:
        cases["poly_negative"] = [type(e).__name__, e.index, e.value]
    # a negative dip narrower than the Gauss-Legendre node spacing: the norm
    # passes, the per-event check fires
    from parafit.pdf import gauss_legendre_points

    gx, _ = gauss_legendre_points(0.0, 1.0, 64, 16)
    c = 0.5 * (gx[500] + gx[501])
    eps = 1e-12
    node3 = polynomial(x, [c * c - eps, -2.0 * c, 1.0])  # (x - c)^2 - eps
    values3 = np.full(7000, 0.9)
    values3[6001] = c
    values3[6500] = c
    ds4 = UnbinnedDataSet([x])
    ds4.extend([values3])
    try:
        nll(node3, ds4)
    except ParafitError as e:
        cases["poly_dip_negative"] = [type(e).__name__, e.index, e.value, c, eps]
    y = Variable.observable("y", 0.0, 10.0)
    g = gaussian(y, Variable("m", 5.0, fixed=True), Variable("s", 0.05, fixed=True))
    e_ = exponential(y, Variable("a", -0.2, fixed=True))
    tree = add_pdf([g, e_], [Variable("f", 1.0, 0.0, 1.0)])  # exponential weight exactly 0
    vals3 = np.full(6000, 5.0)
    vals3[5555] = 9.9  # gaussian underflows to 0 there -> density 0
    ds3 = UnbinnedDataSet([y])
    ds3.extend([vals3])
    try:
        nll(tree, ds3)
    except ParafitError as e:
        cases["sum_underflow"] = [type(e).__name__, e.index, e.value]
    one = UnbinnedDataSet([Variable.observable("z")])
    one.extend([np.array([0.0])])
    z = one.observables[0]
    cases["single_event_gauss"] = nll(gaussian(z, Variable("mu", 0.0, fixed=True), Variable("sg", 1.0, fixed=True)),
                                      one)
    with open(os.path.join(OUT, "errors.json"), "w") as fh:
        json.dump(cases, fh, indent=1)


def fits_fixture():
    """Reference FitManager results (values, errors, minimum, call counts)."""
    from parafit.fitting import FitManager

    out = {}
    g = np.load(os.path.join(OUT, "c1_sumpdf.npz"))
    x, pdf, params = c1_model()
    for v, val in zip(params, (4.8, 0.6, -0.25, 0.35)):
        v.value = val
    ds = UnbinnedDataSet([x])
    ds.extend([g["x"]])
    r = FitManager(pdf, ds).fit()
    out["c1"] = {"start": [4.8, 0.6, -0.25, 0.35], "names": list(r.names), "values": r.values.tolist(),
                 "errors": r.errors.tolist(), "nll_min": r.nll_min, "n_calls": r.n_calls, "status": r.status}
    g2 = np.load(os.path.join(OUT, "c2_prod.npz"))
    x = Variable.observable("x", 0.0, 10.0)
    y = Variable.observable("y", 0.0, 10.0)
    mu = Variable("mu", 4.9, 0.0, 10.0, step=0.01)
    sigma = Variable("sigma", 1.1, 0.01, 5.0, step=1e-3)
    alpha = Variable("alpha", -0.35, -5.0, 5.0, step=1e-3)
    pdf2 = prod_pdf([gaussian(x, mu, sigma), exponential(y, alpha)])
    ds2 = UnbinnedDataSet([x, y])
    ds2.extend([g2["x"], g2["y"]])
    r = FitManager(pdf2, ds2).fit()
    out["c2"] = {"start": [4.9, 1.1, -0.35], "names": list(r.names), "values": r.values.tolist(),
                 "errors": r.errors.tolist(), "nll_min": r.nll_min, "n_calls": r.n_calls, "status": r.status}
    g3 = np.load(os.path.join(OUT, "c3_dalitz.npz"))
    terms = c3_terms()
    start = {"rhom_mag": 0.8, "rhom_ph": 0.05, "rho0_mag": 0.5, "rho0_ph": 0.2, "nr_mag": 18.0, "nr_ph": -0.4}
    for t in terms:
        for var in (t.magnitude, t.phase):
            if var.name in start:
                var.value = start[var.name]
    s12 = Variable.observable("s12", *D_CHANNEL.s12_range)
    s13 = Variable.observable("s13", *D_CHANNEL.s13_range)
    ds3 = UnbinnedDataSet([s12, s13])
    ds3.extend([g3["s12"], g3["s13"]])
    pdf3 = dalitz_pdf(terms, D_CHANNEL, s12_obs=s12, s13_obs=s13, grid=(128, 128))
    r = FitManager(pdf3, ds3).fit()
    out["c3"] = {"start": start, "grid": [128, 128], "names": list(r.names), "values": r.values.tolist(),
                 "errors": r.errors.tolist(), "nll_min": r.nll_min, "n_calls": r.n_calls, "status": r.status}
    with open(os.path.join(OUT, "fits.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def binned_fixture():
    """BinnedDataSet.fill bin contents and binned_nll values / errors / a fit
    (reference core.py:312-379, engine.py:246-276, fitting.py:431-439)."""
    from parafit.core import BinnedDataSet
    from parafit.engine import binned_nll
    from parafit.errors import NonPositiveExpectation
    from parafit.fitting import FitManager

    rng = np.random.default_rng(23)
    out = {}
    # 1-D: the C1 model over 100 bins; data include bin edges and both bounds
    x, pdf, params = c1_model()
    n = 20000
    xs = np.concatenate([np.clip(rng.normal(5.0, 0.5, n // 3), 0, 10), rng.exponential(1 / 0.3, n - n // 3)])
    xs = xs[(xs >= 0) & (xs <= 10)]
    edges = np.array([0.0, 10.0, 0.1, 0.2, 0.3, 0.7, 1.0, 2.5, 9.9, 9.99999999, 5.0, 4.95, 0.30000000000000004])
    xs = np.concatenate([xs, edges])
    ds = UnbinnedDataSet([x])
    ds.extend([xs])
    b1 = BinnedDataSet([x], [100])
    b1.fill(ds)
    out["b1_x"] = xs
    out["b1_contents"] = b1.contents.copy()
    pts1 = [(5.0, 0.5, -0.3, 0.3), (4.8, 0.6, -0.25, 0.35), (5.2, 0.3, -0.5, 0.5)]
    vals = []
    for pt in pts1:
        for v, value in zip(params, pt):
            v.value = value
        vals.append(binned_nll(pdf, b1, snapshot(pdf.param_closure())))
    out["b1_points"] = np.array(pts1)
    out["b1_nll"] = np.array(vals)
    # 2-D: the C2 model over 40 x 25 bins (row-major, y fastest)
    xv = Variable.observable("x", 0.0, 10.0)
    yv = Variable.observable("y", 0.0, 10.0)
    mu = Variable("mu", 5.0, 0.0, 10.0, step=0.01)
    sigma = Variable("sigma", 1.0, 0.01, 5.0, step=1e-3)
    alpha = Variable("alpha", -0.4, -5.0, 5.0, step=1e-3)
    pdf2 = prod_pdf([gaussian(xv, mu, sigma), exponential(yv, alpha)])
    m = 30000
    x2 = np.clip(rng.normal(5.0, 1.0, m), 0, 10)
    y2 = np.clip(rng.exponential(1 / 0.4, m), 0, 10)
    ds2 = UnbinnedDataSet([xv, yv])
    ds2.extend([x2, y2])
    b2 = BinnedDataSet([xv, yv], [40, 25])
    b2.fill(ds2)
    out["b2_x"], out["b2_y"], out["b2_contents"] = x2, y2, b2.contents.copy()
    pts2 = [(5.0, 1.0, -0.4), (4.9, 1.1, -0.35)]
    vals = []
    for pt in pts2:
        mu.value, sigma.value, alpha.value = pt
        vals.append(binned_nll(pdf2, b2, snapshot(pdf2.param_closure())))
    out["b2_points"], out["b2_nll"] = np.array(pts2), np.array(vals)
    mu.value, sigma.value, alpha.value = (4.9, 1.1, -0.35)
    r = FitManager(pdf2, b2).fit()
    out["b2_fit_values"] = np.array(r.values)
    out["b2_fit_errors"] = np.array(r.errors)
    out["b2_fit_nll"] = np.array([r.nll_min])
    out["b2_fit_calls"] = np.array([r.n_calls])
    # NonPositiveExpectation: a narrow gaussian underflows to 0 at far bin centres
    xp = Variable.observable("x", 0.0, 1.0)
    gm = Variable("gm", 0.5, 0.0, 1.0)
    gs = Variable("gs", 0.01, 0.001, 1.0)
    poly = gaussian(xp, gm, gs)
    bp = BinnedDataSet([xp], [20])
    for b in range(20):
        bp.set_content(b, float(b % 3))
    try:
        binned_nll(poly, bp, snapshot(poly.param_closure()))
        raise AssertionError("expected NonPositiveExpectation")
    except NonPositiveExpectation as exc:
        out["bp_contents"] = bp.contents.copy()
        out["bp_bin"] = np.array([exc.bin_index])
        out["bp_value"] = np.array([exc.value])
    except ParafitError as exc:  # the density kernel raised first
        out["bp_contents"] = bp.contents.copy()
        out["bp_error"] = np.array([type(exc).__name__])
    np.savez_compressed(os.path.join(OUT, "binned.npz"), **out)


def toys_fixture():
    """The reference's toy generators (mcgen.py): exact events and stats for a
    few specs, incl. multiple streams and an envelope rescan."""
    from parafit.mcgen import GenSpec as RSpec
    from parafit.mcgen import generate_1d as rgen1d
    from parafit.mcgen import generate_dalitz as rgendal

    out = {}
    x, pdf, params = c1_model()
    for tag, spec in [("a", RSpec(20000, seed=5)), ("b", RSpec(10001, seed=9, streams=3))]:
        stats = {}
        ds = rgen1d(pdf, x, spec, stats)
        out[f"c1{tag}_x"] = ds.column("x")
        out[f"c1{tag}_stats"] = np.array([stats["envelope"], stats["attempts"], stats["accepted"]])
    # a spike the 4096-point scan misses: envelope hit -> rescan -> restart
    xs = Variable.observable("x", 0.0, 10.0)
    spike = gaussian(xs, Variable("m", 5.00061, 0.0, 10.0), Variable("s", 0.001, 1e-5, 1.0))
    stats = {}
    ds = rgen1d(spike, xs, RSpec(300, seed=2, max_attempts_factor=100000), stats)
    out["spike_x"] = ds.column("x")
    out["spike_stats"] = np.array([stats["envelope"], stats["attempts"], stats["accepted"]])
    # ... and one it still misses after the rescan: EnvelopeExceeded
    from parafit.errors import EnvelopeExceeded as REnv

    narrow = gaussian(xs, Variable("m2", 5.00061, 0.0, 10.0), Variable("s2", 0.0005, 1e-5, 1.0))
    try:
        rgen1d(narrow, xs, RSpec(300, seed=2, max_attempts_factor=100000))
        out["narrow_exceeded"] = np.array([0])
    except REnv:
        out["narrow_exceeded"] = np.array([1])
    # the default budget (1000 draws per event) runs out on the spike
    from parafit.errors import AttemptsExhausted as RAtt

    try:
        rgen1d(spike, xs, RSpec(300, seed=2))
        out["spike_exhausted"] = np.array([""])
    except RAtt as exc:
        out["spike_exhausted"] = np.array([str(exc)])
    terms = c3_terms()
    for tag, spec in [("a", RSpec(3000, seed=3)), ("b", RSpec(2001, seed=4, streams=2))]:
        stats = {}
        ds = rgendal(terms, D_CHANNEL, spec, stats=stats)
        out[f"dal{tag}_s12"] = ds.column("s12")
        out[f"dal{tag}_s13"] = ds.column("s13")
        out[f"dal{tag}_stats"] = np.array([stats["envelope"], stats["box_draws"], stats["in_boundary_draws"],
                                           stats["accepted"]])
    np.savez_compressed(os.path.join(OUT, "toys.npz"), **out)


def trees_fixture():
    """NLLs of generic trees (polynomial GL norms, nested add/prod, 3-term sums,
    three observables) from the reference, built from tests/models.TREES."""
    import parafit

    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from tests import models

    out = {}
    for k, (name, spec) in enumerate(models.TREES):
        cols = models.tree_data(name, 3 * 4096 + 321, 100 + k)
        vals = []
        for scale in (0.0, 0.01, -0.02):
            root, obs, _ = models.build_tree(parafit, models.perturb(spec, scale))
            names = sorted(obs)
            ds = UnbinnedDataSet([obs[c] for c in names])
            ds.extend([cols[c] for c in names])
            vals.append(nll(root, ds, snapshot(root.param_closure()), Backend("serial")))
        for c, v in cols.items():
            out[f"{name}__{c}"] = v
        out[f"{name}__nll"] = np.array(vals)
    np.savez_compressed(os.path.join(OUT, "trees.npz"), **out)


def dalitz_variants_fixture():
    """Other Dalitz structures (K = 2, 3, 5; a K pi pi channel with unequal
    masses) -- NLLs at two coefficient points from the reference."""
    import parafit

    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from tests import models

    out = {}
    for k, name in enumerate(sorted(models.DALITZ_VARIANTS)):
        (s12, s13), pdf, terms = models.dalitz_variant(parafit, name)
        ds = generate_dalitz(terms, pdf.payload[1], GenSpec(n_events=2 * 4096 + 321 + k, seed=40 + k),
                             observables=(s12, s13))
        vals = [nll(pdf, ds, snapshot(pdf.param_closure()), Backend("serial"))]
        terms[1].magnitude.value *= 1.1
        terms[-1].phase.value += 0.2
        vals.append(nll(pdf, ds, snapshot(pdf.param_closure()), Backend("serial")))
        out[f"{name}__s12"] = ds.column("s12")
        out[f"{name}__s13"] = ds.column("s13")
        out[f"{name}__nll"] = np.array(vals)
    np.savez_compressed(os.path.join(OUT, "dalitz_variants.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["reduction", "c1", "c2", "c3", "shards", "errors", "fits", "binned", "toys", "trees", "dalitz_variants"]
    for name in which:
        globals()[f"{name}_fixture"]()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
