"""Shared model builders for the tests: the same model as a reference tree
(parafit's own builders -- the API the device engine plugs into) and as an
oracle spec (plain tuples)."""

from __future__ import annotations

import math

import numpy as np
from paper_1710_08826_b200._reference import parafit as P

D_CHANNEL_T = (1.86484, 0.13957, 0.13957, 0.13498)

# (pair, m, width, spin, magnitude, phase) of the C3 D0 -> pi+ pi- pi0 model
C3_TERMS = [
    (13, 0.77511, 0.1491, 1, 1.0, 0.0),
    (23, 0.77511, 0.1491, 1, 0.73, -0.03),
    (12, 0.77526, 0.1478, 1, 0.55, 0.28),
    (12, 1.0, 20.0, 0, 20.0, -0.5),
]


def c1(point=(5.0, 0.5, -0.3, 0.3)):
    pf = ref()
    x = P.Variable.observable("x", 0.0, 10.0)
    mu = P.Variable("mu", point[0], 0.0, 10.0, step=0.01)
    sigma = P.Variable("sigma", point[1], 0.01, 5.0, step=1e-3)
    alpha = P.Variable("alpha", point[2], -5.0, 5.0, step=1e-3)
    f = P.Variable("f", point[3], 0.0, 1.0, step=1e-3)
    pdf = P.add_pdf([P.gaussian(x, mu, sigma), P.exponential(x, alpha)], [f])
    return x, pdf, (mu, sigma, alpha, f)


def c1_spec(point):
    mu, sigma, alpha, f = point
    return ("add", [("gaussian", "x", mu, sigma, 0.0, 10.0), ("exponential", "x", alpha, 0.0, 10.0)], [f])


def c2(point=(5.0, 1.0, -0.4)):
    pf = ref()
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    mu = P.Variable("mu", point[0], 0.0, 10.0, step=0.01)
    sigma = P.Variable("sigma", point[1], 0.01, 5.0, step=1e-3)
    alpha = P.Variable("alpha", point[2], -5.0, 5.0, step=1e-3)
    pdf = P.prod_pdf([P.gaussian(x, mu, sigma), P.exponential(y, alpha)])
    return (x, y), pdf, (mu, sigma, alpha)


def c2_spec(point):
    mu, sigma, alpha = point
    return ("prod", [("gaussian", "x", mu, sigma, 0.0, 10.0), ("exponential", "y", alpha, 0.0, 10.0)])


def c3(terms=C3_TERMS, grid=(400, 400)):
    pf = ref()
    ch = P.DecayChannel(*D_CHANNEL_T)
    rts = []
    for k, (pair, m, w, spin, mag, ph) in enumerate(terms):
        rts.append(P.ResonanceTerm(
            pair=pair,
            mass=P.Variable(f"t{k}_m", m, fixed=True),
            width=P.Variable(f"t{k}_w", w, fixed=True),
            spin=spin,
            magnitude=P.Variable(f"t{k}_mag", mag, 0.0, 100.0, step=0.01, fixed=(k == 0)),
            phase=P.Variable(f"t{k}_ph", ph, -2 * math.pi, 2 * math.pi, step=0.01, fixed=(k == 0)),
        ))
    s12 = P.Variable.observable("s12", *ch.s12_range)
    s13 = P.Variable.observable("s13", *ch.s13_range)
    pdf = P.dalitz_pdf(rts, ch, s12_obs=s12, s13_obs=s13, grid=grid)
    return (s12, s13), pdf, rts


def c3_spec(terms=C3_TERMS, grid=(400, 400)):
    spec_terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in terms]
    return ("dalitz", "s12", "s13", spec_terms, D_CHANNEL_T, grid)


def ref():
    """The reference package (parafit) the engine plugs into."""
    from paper_1710_08826_b200._reference import parafit

    return parafit


def dataset(observables, columns):
    """A DeviceDataSet (a reference UnbinnedDataSet) over whole columns; the
    HBM copy is made on the first device NLL."""
    from paper_1710_08826_b200.datasets import DeviceDataSet

    return DeviceDataSet.from_columns(list(observables), [np.asarray(c, dtype=np.float64) for c in columns],
                                      device=None)


def ref_dataset(observables, columns):
    """The reference's own list-backed UnbinnedDataSet (small inputs only)."""
    ds = ref().UnbinnedDataSet(list(observables))
    ds.extend([np.asarray(c, dtype=np.float64) for c in columns])
    return ds


# --- generic trees: one spec language for the reference, this package and the oracle ---

TREE_OBS = {"x": (0.0, 10.0), "y": (-2.0, 3.0), "z": (0.0, 1.0), "w": (1.0, 4.0)}

# (name, spec) -- leaf specs are the oracle's: ("gaussian", col, mu, sigma, lo, hi),
# ("exponential", col, alpha, lo, hi), ("polynomial", col, coeffs, lo, hi);
# ("add", [children], [fractions]), ("prod", [children])
def _g(c, mu, s):
    return ("gaussian", c, mu, s) + TREE_OBS[c]


def _e(c, a):
    return ("exponential", c, a) + TREE_OBS[c]


def _p(c, coeffs):
    return ("polynomial", c, list(coeffs)) + TREE_OBS[c]


TREES = [
    ("gauss_poly", ("add", [_g("x", 4.0, 1.2), _p("x", [1.0, 0.2, 0.03])], [0.4])),
    ("sum_times_poly", ("prod", [("add", [_g("x", 5.0, 0.7), _e("x", -0.2)], [0.6]), _p("y", [2.0, 0.1])])),
    ("sum_of_prods", ("add", [("prod", [_g("x", 6.0, 1.5), _g("y", 0.5, 0.8)]),
                              ("prod", [_e("x", -0.3), _p("y", [1.0, 0.2])])], [0.35])),
    ("three_terms", ("add", [_g("x", 3.0, 0.5), _e("x", -0.15), _p("x", [1.0, -0.05])], [0.3, 0.25])),
    ("prod3", ("prod", [_g("x", 5.5, 2.0), _e("y", 0.3), _p("z", [0.5, 1.0, 0.2])])),
    ("prod4", ("prod", [("add", [_g("x", 5.0, 1.0), _e("x", -0.1)], [0.5]), _e("y", 0.2), _p("z", [0.5, 1.0]),
                        _g("w", 2.5, 0.6)])),
    ("gauss", _g("x", 4.5, 1.1)),
    ("expo", _e("x", -0.25)),
    ("poly", _p("z", [0.3, 0.0, 2.0, 0.5])),
]


def tree_columns(spec, out=None):
    out = set() if out is None else out
    if spec[0] in ("add", "prod"):
        for ch in spec[1]:
            tree_columns(ch, out)
    else:
        out.add(spec[1])
    return out


def build_tree(mod, spec, obs=None, params=None):
    """The spec as a PdfNode tree of `mod` (the reference package or this one:
    the builders have the same names).  Returns (root, observables, params)."""
    obs = {} if obs is None else obs
    params = [] if params is None else params

    def var_obs(c):
        if c not in obs:
            obs[c] = mod.Variable.observable(c, *TREE_OBS[c])
        return obs[c]

    def par(name, v, lo, hi):
        p = mod.Variable(f"{name}{len(params)}", v, lo, hi)
        params.append(p)
        return p

    k = spec[0]
    if k == "gaussian":
        node = mod.gaussian(var_obs(spec[1]), par("mu", spec[2], -20.0, 20.0), par("sg", spec[3], 1e-3, 50.0))
    elif k == "exponential":
        node = mod.exponential(var_obs(spec[1]), par("al", spec[2], -10.0, 10.0))
    elif k == "polynomial":
        node = mod.polynomial(var_obs(spec[1]), [par("c", c, -10.0, 10.0) for c in spec[2]])
    elif k == "add":
        kids = [build_tree(mod, ch, obs, params)[0] for ch in spec[1]]
        node = mod.add_pdf(kids, [par("f", f, 0.0, 1.0) for f in spec[2]])
    else:
        node = mod.prod_pdf([build_tree(mod, ch, obs, params)[0] for ch in spec[1]])
    return node, obs, params


def perturb(spec, scale):
    """The spec with every parameter multiplied by (1 + scale) (fractions too)."""
    k = spec[0]
    if k == "add":
        return ("add", [perturb(ch, scale) for ch in spec[1]], [f * (1 + scale) for f in spec[2]])
    if k == "prod":
        return ("prod", [perturb(ch, scale) for ch in spec[1]])
    if k == "polynomial":
        return (k, spec[1], [c * (1 + scale) for c in spec[2]]) + tuple(spec[3:])
    if k == "gaussian":
        return (k, spec[1], spec[2] * (1 + scale), spec[3] * (1 + scale)) + tuple(spec[4:])
    return (k, spec[1], spec[2] * (1 + scale)) + tuple(spec[3:])


def tree_data(name, n, seed):
    """Uniform events over the spec's observables (deterministic per tree)."""
    rng = np.random.default_rng(seed)
    spec = dict(TREES)[name]
    cols = {}
    for c in sorted(tree_columns(spec)):
        lo, hi = TREE_OBS[c]
        cols[c] = rng.uniform(lo, hi, n)
    return cols


# --- Dalitz variants (kernel dispatch coverage: K = 2, 3, 4 other structures, 5) ----

DALITZ_VARIANTS = {
    # name: (channel (M, m1, m2, m3), [(pair, m, width, spin, mag, phase)], grid)
    "k2": ((1.86484, 0.13957, 0.13957, 0.13498),
           [(13, 0.77511, 0.1491, 1, 1.0, 0.0), (12, 1.0, 20.0, 0, 15.0, -0.5)], (96, 96)),
    "k3": ((1.86484, 0.13957, 0.13957, 0.13498),
           [(13, 0.77511, 0.1491, 1, 1.0, 0.0), (23, 0.77511, 0.1491, 1, 0.73, -0.03),
            (12, 0.77526, 0.1478, 1, 0.55, 0.28)], (96, 96)),
    "k4_kpipi": ((1.86966, 0.493677, 0.13957, 0.13957),
                 [(12, 0.89555, 0.0473, 1, 1.0, 0.0), (13, 0.89555, 0.0473, 1, 1.0, 0.3),
                  (23, 0.98, 0.07, 0, 2.0, 1.2), (12, 1.425, 0.27, 0, 1.5, -0.7)], (96, 96)),
    "k5": ((1.86484, 0.13957, 0.13957, 0.13498),
           [(13, 0.77511, 0.1491, 1, 1.0, 0.0), (23, 0.77511, 0.1491, 1, 0.73, -0.03),
            (12, 0.77526, 0.1478, 1, 0.55, 0.28), (12, 1.0, 20.0, 0, 20.0, -0.5),
            (13, 1.465, 0.4, 1, 0.4, 2.0)], (96, 96)),
}


def dalitz_variant(mod, name):
    """(observables, pdf, terms) of a variant with `mod`'s builders (the
    reference package or this one)."""
    ch_t, spec, grid = DALITZ_VARIANTS[name]
    ch = mod.DecayChannel(*ch_t)
    terms = []
    for k, (pair, m, w, spin, mag, ph) in enumerate(spec):
        terms.append(mod.ResonanceTerm(
            pair=pair, mass=mod.Variable(f"{name}{k}_m", m, fixed=True),
            width=mod.Variable(f"{name}{k}_w", w, fixed=True), spin=spin,
            magnitude=mod.Variable(f"{name}{k}_mag", mag, 0.0, 100.0, fixed=(k == 0)),
            phase=mod.Variable(f"{name}{k}_ph", ph, -2 * math.pi, 2 * math.pi, fixed=(k == 0))))
    s12 = mod.Variable.observable("s12", *ch.s12_range)
    s13 = mod.Variable.observable("s13", *ch.s13_range)
    pdf = mod.dalitz_pdf(terms, ch, s12_obs=s12, s13_obs=s13, grid=grid)
    return (s12, s13), pdf, terms
