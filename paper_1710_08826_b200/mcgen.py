"""Synthetic event generation for benchmarks and tests (host numpy).

Not on the NLL path: these samplers only produce the input columns.  The
reference generates by PCG64 accept-reject (mcgen.py:68-257); parity never
depends on the sampler because the device and the CPU reference always
consume the same arrays.  Samplers here are exact inverse-CDF where a closed
form exists (truncated exponential, truncated Gaussian via erf/erfinv-free
accept on a wide proposal) and vectorised accept-reject for the Dalitz plot.
"""

from __future__ import annotations

import math

import numpy as np


def truncated_gaussian(n: int, mu: float, sigma: float, lo: float, hi: float, rng) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    got = 0
    while got < n:
        k = int((n - got) * 1.2) + 1024
        v = rng.normal(mu, sigma, k)
        v = v[(v >= lo) & (v <= hi)]
        take = min(len(v), n - got)
        out[got:got + take] = v[:take]
        got += take
    return out


def truncated_exponential(n: int, alpha: float, lo: float, hi: float, rng) -> np.ndarray:
    """Inverse CDF of exp(alpha x) on [lo, hi]."""
    u = rng.random(n)
    if alpha == 0.0:
        return lo + (hi - lo) * u
    a, b = math.exp(alpha * lo), math.exp(alpha * hi)
    x = np.log(a + u * (b - a)) / alpha
    return np.clip(x, lo, hi)


def sumpdf_1d(n: int, mu: float, sigma: float, alpha: float, f: float, lo: float, hi: float, seed: int):
    """C1 / C5: f * Gauss + (1 - f) * Exp on [lo, hi]."""
    rng = np.random.default_rng(seed)
    ng = int(rng.binomial(n, f))
    x = np.concatenate([truncated_gaussian(ng, mu, sigma, lo, hi, rng),
                        truncated_exponential(n - ng, alpha, lo, hi, rng)])
    rng.shuffle(x)
    return x


def prod_2d(n: int, mu: float, sigma: float, alpha: float, lo: float, hi: float, seed: int):
    """C2: x ~ Gauss(mu, sigma), y ~ Exp(alpha), independent, on [lo, hi]^2."""
    rng = np.random.default_rng(seed)
    return truncated_gaussian(n, mu, sigma, lo, hi, rng), truncated_exponential(n, alpha, lo, hi, rng)


def _boundary(s12, s13, M, m1, m2, m3):
    with np.errstate(invalid="ignore", divide="ignore"):
        rs = np.sqrt(s12)
        e1 = (s12 + m1 * m1 - m2 * m2) / (2.0 * rs)
        e3 = (M * M - s12 - m3 * m3) / (2.0 * rs)
        p1 = np.sqrt(e1 * e1 - m1 * m1)
        p3 = np.sqrt(e3 * e3 - m3 * m3)
        es = (e1 + e3) ** 2
        return (s13 >= es - (p1 + p3) ** 2) & (s13 <= es - (p1 - p3) ** 2)


def _intensity(terms, s12, s13, M, m1, m2, m3):
    mss = M * M + m1 * m1 + m2 * m2 + m3 * m3
    s23 = mss - s12 - s13
    tot = 0j
    for pair, spin, m, w, mag, ph in terms:
        s = s12 if pair == 12 else (s13 if pair == 13 else s23)
        a = 1.0 / (m * m - s - 1j * m * w)
        if spin == 1:
            if pair == 12:
                z = s13 - s23 + (M * M - m3 * m3) * (m2 * m2 - m1 * m1) / s12
            elif pair == 13:
                z = s12 - s23 + (M * M - m2 * m2) * (m3 * m3 - m1 * m1) / s13
            else:
                z = s12 - s13 + (M * M - m1 * m1) * (m3 * m3 - m2 * m2) / s23
            a = a * z
        tot = tot + mag * np.exp(1j * ph) * a
    return (tot * np.conj(tot)).real


def dalitz(n: int, terms, channel, seed: int, chunk: int = 1 << 22):
    """Accept-reject over the (s12, s13) box; terms = [(pair, spin, m, w, mag, phase)]."""
    M, m1, m2, m3 = channel
    lo12, hi12 = (m1 + m2) ** 2, (M - m3) ** 2
    lo13, hi13 = (m1 + m3) ** 2, (M - m2) ** 2
    rng = np.random.default_rng(seed)
    g12 = lo12 + (np.arange(512) + 0.5) * (hi12 - lo12) / 512
    g13 = lo13 + (np.arange(512) + 0.5) * (hi13 - lo13) / 512
    G12, G13 = np.meshgrid(g12, g13, indexing="ij")
    inside = _boundary(G12, G13, M, m1, m2, m3)
    env = 1.2 * float(_intensity(terms, G12[inside], G13[inside], M, m1, m2, m3).max())
    a12, a13 = np.empty(n), np.empty(n)
    got = 0
    while got < n:
        c12 = rng.uniform(lo12, hi12, chunk)
        c13 = rng.uniform(lo13, hi13, chunk)
        ok = _boundary(c12, c13, M, m1, m2, m3)
        c12, c13 = c12[ok], c13[ok]
        keep = rng.uniform(0.0, env, len(c12)) < _intensity(terms, c12, c13, M, m1, m2, m3)
        c12, c13 = c12[keep], c13[keep]
        take = min(len(c12), n - got)
        a12[got:got + take] = c12[:take]
        a13[got:got + take] = c13[:take]
        got += take
    return a12, a13


# --- device generation (libpfb200: pfb_gen_1d / pfb_gen_dalitz) -------------------------


def _device_store(ctx, ncols: int, n: int):
    import ctypes

    from . import _lib as L

    st = ctypes.c_void_p()
    L.check(L.lib().pfb_store_create(ctx.handle, ncols, n, ctypes.byref(st)), "pfb_store_create")
    return st


def _adopt(ctx, st, ncols: int, n: int):
    """Download the generated columns and register the device store as the
    HBM copy of those host arrays (no re-upload when the NLL runs)."""
    from . import _lib as L

    cols = []
    for c in range(ncols):
        a = np.empty(n, dtype=np.float64)
        L.check(L.lib().pfb_store_download(st, c, L.dptr(a), 0, n), "pfb_store_download")
        cols.append(a)
    ctx._stores[tuple(id(a) for a in cols) + (0, n)] = (st, tuple(cols))
    return cols


def device_sumpdf_1d(n, mu, sigma, alpha, f, lo, hi, seed, ctx=None):
    """C1 / C5 events generated on the GPU: f * Gauss + (1 - f) * Exp on [lo, hi]."""
    from . import _lib as L
    from .engine import device_context

    ctx = ctx or device_context(0)
    st = _device_store(ctx, 1, n)
    L.check(L.lib().pfb_gen_1d(ctx.handle, 0, mu, sigma, alpha, f, lo, hi, seed, n, st), "pfb_gen_1d")
    return _adopt(ctx, st, 1, n)[0]


def device_prod_2d(n, mu, sigma, alpha, lo, hi, seed, ctx=None):
    """C2 events generated on the GPU: Gauss(x) x Exp(y) on [lo, hi]^2."""
    from . import _lib as L
    from .engine import device_context

    ctx = ctx or device_context(0)
    st = _device_store(ctx, 2, n)
    L.check(L.lib().pfb_gen_1d(ctx.handle, 1, mu, sigma, alpha, 0.0, lo, hi, seed, n, st), "pfb_gen_1d")
    return tuple(_adopt(ctx, st, 2, n))


def dalitz_envelope(terms, channel, safety: float = 1.2, points: int = 512) -> float:
    """safety x the largest intensity on a points^2 midpoint scan (reference mcgen.py:180-181)."""
    M, m1, m2, m3 = channel
    lo12, hi12 = (m1 + m2) ** 2, (M - m3) ** 2
    lo13, hi13 = (m1 + m3) ** 2, (M - m2) ** 2
    g12 = lo12 + (np.arange(points) + 0.5) * (hi12 - lo12) / points
    g13 = lo13 + (np.arange(points) + 0.5) * (hi13 - lo13) / points
    G12, G13 = np.meshgrid(g12, g13, indexing="ij")
    inside = _boundary(G12, G13, M, m1, m2, m3)
    return safety * float(_intensity(terms, G12[inside], G13[inside], M, m1, m2, m3).max())


def device_dalitz(n, terms, channel, seed, ctx=None, envelope=None):
    """Dalitz events generated on the GPU; terms = [(pair, spin, m, w, mag, phase)]."""
    import ctypes

    from . import _lib as L
    from .engine import device_context

    ctx = ctx or device_context(0)
    d = L.PfbDalitzDesc()
    d.mother_mass, d.m1, d.m2, d.m3 = channel
    d.nterms = len(terms)
    vals = np.zeros(4 * len(terms))
    for k, (pair, spin, m, w, mag, ph) in enumerate(terms):
        d.pair[k], d.spin[k] = int(pair), int(spin)
        vals[4 * k:4 * k + 4] = (m, w, mag, ph)
    env = envelope if envelope is not None else dalitz_envelope(terms, channel)
    st = _device_store(ctx, 2, n)
    cand = ctypes.c_int64()
    L.check(L.lib().pfb_gen_dalitz(ctx.handle, ctypes.byref(d), L.dptr(vals), env, seed, n, st, ctypes.byref(cand)),
            "pfb_gen_dalitz")
    return tuple(_adopt(ctx, st, 2, n))
