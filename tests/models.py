"""Shared model builders for the tests: the same model as a device tree
(paper_1710_08826_b200 nodes) and as an oracle spec (plain tuples)."""

from __future__ import annotations

import math

import numpy as np

D_CHANNEL_T = (1.86484, 0.13957, 0.13957, 0.13498)

# (pair, m, width, spin, magnitude, phase) of the C3 D0 -> pi+ pi- pi0 model
C3_TERMS = [
    (13, 0.77511, 0.1491, 1, 1.0, 0.0),
    (23, 0.77511, 0.1491, 1, 0.73, -0.03),
    (12, 0.77526, 0.1478, 1, 0.55, 0.28),
    (12, 1.0, 20.0, 0, 20.0, -0.5),
]


def c1(point=(5.0, 0.5, -0.3, 0.3)):
    import paper_1710_08826_b200 as pf

    x = pf.Variable.observable("x", 0.0, 10.0)
    mu = pf.Variable("mu", point[0], 0.0, 10.0, step=0.01)
    sigma = pf.Variable("sigma", point[1], 0.01, 5.0, step=1e-3)
    alpha = pf.Variable("alpha", point[2], -5.0, 5.0, step=1e-3)
    f = pf.Variable("f", point[3], 0.0, 1.0, step=1e-3)
    pdf = pf.add_pdf([pf.gaussian(x, mu, sigma), pf.exponential(x, alpha)], [f])
    return x, pdf, (mu, sigma, alpha, f)


def c1_spec(point):
    mu, sigma, alpha, f = point
    return ("add", [("gaussian", "x", mu, sigma, 0.0, 10.0), ("exponential", "x", alpha, 0.0, 10.0)], [f])


def c2(point=(5.0, 1.0, -0.4)):
    import paper_1710_08826_b200 as pf

    x = pf.Variable.observable("x", 0.0, 10.0)
    y = pf.Variable.observable("y", 0.0, 10.0)
    mu = pf.Variable("mu", point[0], 0.0, 10.0, step=0.01)
    sigma = pf.Variable("sigma", point[1], 0.01, 5.0, step=1e-3)
    alpha = pf.Variable("alpha", point[2], -5.0, 5.0, step=1e-3)
    pdf = pf.prod_pdf([pf.gaussian(x, mu, sigma), pf.exponential(y, alpha)])
    return (x, y), pdf, (mu, sigma, alpha)


def c2_spec(point):
    mu, sigma, alpha = point
    return ("prod", [("gaussian", "x", mu, sigma, 0.0, 10.0), ("exponential", "y", alpha, 0.0, 10.0)])


def c3(terms=C3_TERMS, grid=(400, 400)):
    import paper_1710_08826_b200 as pf

    ch = pf.DecayChannel(*D_CHANNEL_T)
    rts = []
    for k, (pair, m, w, spin, mag, ph) in enumerate(terms):
        rts.append(pf.ResonanceTerm(
            pair=pair,
            mass=pf.Variable(f"t{k}_m", m, fixed=True),
            width=pf.Variable(f"t{k}_w", w, fixed=True),
            spin=spin,
            magnitude=pf.Variable(f"t{k}_mag", mag, 0.0, 100.0, step=0.01, fixed=(k == 0)),
            phase=pf.Variable(f"t{k}_ph", ph, -2 * math.pi, 2 * math.pi, step=0.01, fixed=(k == 0)),
        ))
    s12 = pf.Variable.observable("s12", *ch.s12_range)
    s13 = pf.Variable.observable("s13", *ch.s13_range)
    pdf = pf.dalitz_pdf(rts, ch, s12_obs=s12, s13_obs=s13, grid=grid)
    return (s12, s13), pdf, rts


def c3_spec(terms=C3_TERMS, grid=(400, 400)):
    spec_terms = [(p, s, m, w, mag, ph) for (p, m, w, s, mag, ph) in terms]
    return ("dalitz", "s12", "s13", spec_terms, D_CHANNEL_T, grid)


def dataset(observables, columns):
    import paper_1710_08826_b200 as pf

    ds = pf.UnbinnedDataSet(list(observables))
    ds.extend([np.asarray(c, dtype=np.float64) for c in columns])
    return ds
