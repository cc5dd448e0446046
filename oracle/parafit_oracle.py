"""CPU oracle for the NLL hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (parafit, /root/reference/
pkg/src/parafit) for the per-event PDF evaluation and the NLL reduction.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module; the product path never does.

Pinned against the real reference: tests/golden/make_golden.py imports the
reference from /root/reference (in the build container) and records its
outputs; tests/test_oracle.py checks this module against those fixtures
(bit-exact for block sums, shard bounds, grid masks; 0 ulp on NLLs computed
with the same numpy ops).

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK = 4096  # reduction.py:25


class OracleDensityError(Exception):
    """A density check failed: kind in {NonPositiveDensity, NonFiniteDensity,
    NegativeDensity, FractionOutOfRange, EmptyDataSet}."""

    def __init__(self, kind: str, index: int = -1, value: float = float("nan")):
        self.kind, self.index, self.value = kind, index, value
        super().__init__(f"{kind}(index={index}, value={value!r})")


# --- reduction (reduction.py) --------------------------------------------------------


def fold_halves_matrix(mat: np.ndarray) -> np.ndarray:
    """reduction.py:28-42: pair j with j + width/2 at every level."""
    while mat.shape[1] > 1:
        half = mat.shape[1] // 2
        mat = mat[:, :half] + mat[:, half:]
    return mat[:, 0]


def pairwise_sum_1d(a) -> float:
    """reduction.py:45-56: split recursion, <= 8 leaves summed left to right."""
    n = len(a)
    if n == 0:
        return 0.0
    if n <= 8:
        s = float(a[0])
        for k in range(1, n):
            s += float(a[k])
        return s
    half = n // 2
    return pairwise_sum_1d(a[:half]) + pairwise_sum_1d(a[half:])


def block_sums(terms: np.ndarray, block: int = BLOCK) -> np.ndarray:
    """reduction.py:59-75."""
    n = len(terms)
    n_full = n // block
    out = np.empty(n_full + (1 if n % block else 0), dtype=np.float64)
    if n_full:
        out[:n_full] = fold_halves_matrix(terms[: n_full * block].reshape(n_full, block))
    if n % block:
        out[n_full] = pairwise_sum_1d(terms[n_full * block:])
    return out


def exact_total(values) -> float:
    """engine.py:240-243 / reduction.py:127-137: correctly rounded sum."""
    return math.fsum(list(values))


def shard_bounds(n: int, workers: int, block: int = BLOCK) -> list[int]:
    """sharding.py:80-85."""
    base, extra = divmod(n, workers)
    bounds = [0]
    for k in range(workers):
        bounds.append(bounds[-1] + base + (1 if k < extra else 0))
    if n >= workers * block:
        bounds = [0] + [(b // block) * block for b in bounds[1:-1]] + [n]
    return bounds


def chunk_ranges(n_events: int, workers: int, block: int = BLOCK):
    """engine.py:74-92 (pool mode)."""
    n_blocks = -(-n_events // block)
    n_chunks = min(workers, n_blocks)
    if n_chunks <= 0:
        return []
    base, extra = divmod(n_blocks, n_chunks)
    ranges, b0 = [], 0
    for k in range(n_chunks):
        b1 = b0 + base + (1 if k < extra else 0)
        if b1 > b0:
            ranges.append((b0 * block, min(b1 * block, n_events)))
        b0 = b1
    return ranges


# --- primitive densities and norms (pdf.py) ---------------------------------------------


def _check_finite(values, index_base=0):
    bad = ~np.isfinite(values)
    if bad.any():
        raise OracleDensityError("NonFiniteDensity", int(np.argmax(bad)))
    return values


def gaussian_kernel(x, mu, sigma):
    """pdf.py:122-127."""
    z = (x - mu) / sigma
    return _check_finite(np.exp(-0.5 * z * z))


def exponential_kernel(x, alpha):
    """pdf.py:141-144."""
    return _check_finite(np.exp(alpha * x))


def polynomial_kernel(x, coeffs):
    """pdf.py:164-178 (np.polynomial.polynomial.polyval = Horner)."""
    vals = np.asarray(np.polynomial.polynomial.polyval(x, np.asarray(coeffs, dtype=np.float64)), dtype=np.float64)
    _check_finite(vals)
    neg = vals < 0.0
    if neg.any():
        i = int(np.argmax(neg))
        raise OracleDensityError("NegativeDensity", i, float(vals[i]))
    return vals


def gaussian_norm(mu, sigma, lo, hi):
    """pdf.py:130-138."""
    s2 = math.sqrt(2.0)
    h = math.erf((hi - mu) / (sigma * s2)) if not math.isinf(hi) else 1.0
    l = math.erf((lo - mu) / (sigma * s2)) if not math.isinf(lo) else -1.0
    return sigma * math.sqrt(0.5 * math.pi) * (h - l)


def exponential_norm(alpha, lo, hi):
    """pdf.py:147-161 (finite bounds)."""
    if alpha == 0.0:
        return hi - lo
    return (math.exp(alpha * hi) - math.exp(alpha * lo)) / alpha


def gl_points(lo, hi, nodes=64, panels=16):
    """pdf.py:181-189."""
    xi, wi = np.polynomial.legendre.leggauss(nodes)
    width = (hi - lo) / panels
    starts = lo + width * np.arange(panels)
    centers = starts + 0.5 * width
    x = (centers[:, None] + 0.5 * width * xi[None, :]).reshape(-1)
    w = np.broadcast_to(0.5 * width * wi, (panels, nodes)).reshape(-1)
    return x, w


def polynomial_norm(coeffs, lo, hi, nodes=64, panels=16):
    """pdf.py:192-199."""
    x, w = gl_points(lo, hi, nodes, panels)
    return float(np.dot(w, polynomial_kernel(x, coeffs)))


# --- Dalitz (dalitz.py) ---------------------------------------------------------------------


def s13_limits(s12, M, m1, m2, m3):
    """dalitz.py:127-140."""
    s12 = np.asarray(s12, dtype=np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        rs = np.sqrt(s12)
        e1 = (s12 + m1**2 - m2**2) / (2.0 * rs)
        e3 = (M**2 - s12 - m3**2) / (2.0 * rs)
        p1 = np.sqrt(e1 * e1 - m1**2)
        p3 = np.sqrt(e3 * e3 - m3**2)
        esum = (e1 + e3) ** 2
        return esum - (p1 + p3) ** 2, esum - (p1 - p3) ** 2


def in_boundary_mask(s12, s13, M, m1, m2, m3):
    """dalitz.py:143-150."""
    s12 = np.asarray(s12, dtype=np.float64)
    s13 = np.asarray(s13, dtype=np.float64)
    lo12, hi12 = (m1 + m2) ** 2, (M - m3) ** 2
    lo, hi = s13_limits(s12, M, m1, m2, m3)
    with np.errstate(invalid="ignore"):
        return (s12 >= lo12) & (s12 <= hi12) & (s13 >= lo) & (s13 <= hi)


def integration_grid(M, m1, m2, m3, grid=(400, 400)):
    """dalitz.py:246-264."""
    nx, ny = grid
    lo12, hi12 = (m1 + m2) ** 2, (M - m3) ** 2
    lo13, hi13 = (m1 + m3) ** 2, (M - m2) ** 2
    dx = (hi12 - lo12) / nx
    dy = (hi13 - lo13) / ny
    g12, g13 = np.meshgrid(lo12 + (np.arange(nx) + 0.5) * dx, lo13 + (np.arange(ny) + 0.5) * dy, indexing="ij")
    g12, g13 = g12.reshape(-1), g13.reshape(-1)
    return g12, g13, in_boundary_mask(g12, g13, M, m1, m2, m3), dx * dy


def amplitude_values(pair, spin, m, width, s12, s13, M, m1, m2, m3):
    """dalitz.py:162-197 (BW x Zemach spin-1 factor)."""
    s12 = np.asarray(s12, dtype=np.float64)
    s13 = np.asarray(s13, dtype=np.float64)
    mss = M**2 + m1**2 + m2**2 + m3**2
    s23 = mss - s12 - s13
    s = s12 if pair == 12 else (s13 if pair == 13 else s23)
    bw = 1.0 / (m * m - s - 1j * (m * width))
    if spin == 1:
        M2, m1sq, m2sq, m3sq = M**2, m1**2, m2**2, m3**2
        if pair == 12:
            z = s13 - s23 + (M2 - m3sq) * (m2sq - m1sq) / s12
        elif pair == 13:
            z = s12 - s23 + (M2 - m2sq) * (m3sq - m1sq) / s13
        else:
            z = s12 - s13 + (M2 - m1sq) * (m3sq - m2sq) / s23
        bw = bw * z
    return bw


def coefficients(terms):
    """dalitz.py:211-214; terms = [(pair, spin, m, w, mag, phase)]."""
    mags = np.array([t[4] for t in terms], dtype=np.float64)
    phases = np.array([t[5] for t in terms], dtype=np.float64)
    return mags * np.exp(1j * phases)


def intensity_values(terms, s12, s13, channel):
    """dalitz.py:217-230."""
    c = coefficients(terms)
    total = None
    for ck, t in zip(c, terms):
        contrib = ck * amplitude_values(t[0], t[1], t[2], t[3], s12, s13, *channel)
        total = contrib if total is None else total + contrib
    return (total * np.conj(total)).real


def compute_integrals(terms, channel, grid=(400, 400)):
    """dalitz.py:282-329 (no prior)."""
    g12, g13, mask, darea = integration_grid(*channel, grid)
    p12, p13 = g12[mask], g13[mask]
    n = len(terms)
    amps = np.empty((n, p12.size), dtype=np.complex128)
    for i, t in enumerate(terms):
        amps[i] = amplitude_values(t[0], t[1], t[2], t[3], p12, p13, *channel)
    mat = np.empty((n, n), dtype=np.complex128)
    for i in range(n):
        for j in range(i, n):
            if i == j:
                re, im = amps[i].real, amps[i].imag
                val = complex(float(np.sum(re * re + im * im)) * darea, 0.0)
            else:
                val = np.sum(amps[i] * np.conj(amps[j])) * darea
            mat[i, j] = val
            mat[j, i] = val.conjugate()
    return mat


def dalitz_norm(terms, matrix):
    """dalitz.py:332-349."""
    c = coefficients(terms)
    return complex(np.dot(c, matrix @ np.conj(c))).real


# --- model specs and the NLL ---------------------------------------------------------------
#
# A spec is a plain nested tuple, independent of any package's classes:
#   ("gaussian", col, mu, sigma, lo, hi) | ("exponential", col, alpha, lo, hi)
#   ("polynomial", col, coeffs, lo, hi) | ("add", [children], [fractions])
#   ("prod", [children]) | ("dalitz", col12, col13, terms, channel, grid)


def spec_norm(spec, dalitz_matrix=None) -> float:
    k = spec[0]
    if k == "gaussian":
        return gaussian_norm(spec[2], spec[3], spec[4], spec[5])
    if k == "exponential":
        return exponential_norm(spec[2], spec[3], spec[4])
    if k == "polynomial":
        return polynomial_norm(spec[2], spec[3], spec[4])
    if k in ("add", "prod"):
        return 1.0
    if k == "dalitz":
        mat = dalitz_matrix if dalitz_matrix is not None else compute_integrals(spec[3], spec[4], spec[5])
        return dalitz_norm(spec[3], mat)
    raise ValueError(k)


def spec_eval(spec, cols, cache=None):
    """eval_batch recursion (pdf.py:251-269, 205-227)."""
    k = spec[0]
    if k == "gaussian":
        return gaussian_kernel(cols[spec[1]], spec[2], spec[3])
    if k == "exponential":
        return exponential_kernel(cols[spec[1]], spec[2])
    if k == "polynomial":
        return polynomial_kernel(cols[spec[1]], spec[2])
    if k == "add":
        f = np.array(spec[2], dtype=np.float64)
        rest = 1.0 - f.sum()
        if (f < 0.0).any() or (f > 1.0).any() or rest < 0.0:
            raise OracleDensityError("FractionOutOfRange")
        weights = np.append(f, rest)
        total = None
        for w, child in zip(weights, spec[1]):
            dens = spec_eval(child, cols, cache) / spec_norm_cached(child, cache)
            total = w * dens if total is None else total + w * dens
        return total
    if k == "prod":
        total = None
        for child in spec[1]:
            dens = spec_eval(child, cols, cache) / spec_norm_cached(child, cache)
            total = dens if total is None else total * dens
        return total
    if k == "dalitz":
        return intensity_values(spec[3], cols[spec[1]], cols[spec[2]], spec[4])
    raise ValueError(k)


def spec_norm_cached(spec, cache):
    if cache is None:
        return spec_norm(spec)
    key = id(spec)
    if key not in cache:
        cache[key] = spec_norm(spec)
    return cache[key]


def nll_terms(spec, cols, start, stop, offset=0, cache=None):
    """engine.py:170-187."""
    sliced = {name: c[start:stop] for name, c in cols.items()}
    dens = spec_eval(spec, sliced, cache)
    p = dens / spec_norm_cached(spec, cache)
    good = p > 0.0
    if not good.all():
        i = int(np.argmax(~good))
        raise OracleDensityError("NonPositiveDensity", offset + start + i, float(p[i]))
    return -np.log(p)


def nll(spec, cols, workers: int = 1, block: int = BLOCK) -> float:
    """engine.py:214-243 with the serial (workers=1) or pool backend."""
    n = len(next(iter(cols.values())))
    if n == 0:
        raise OracleDensityError("EmptyDataSet")
    cache: dict = {}
    spec_norm_cached(spec, cache)
    ranges = [(0, n)] if workers == 1 else chunk_ranges(n, workers, block)

    def one(r):
        return block_sums(nll_terms(spec, cols, r[0], r[1], 0, cache), block)

    if workers == 1:
        chunks = [one(r) for r in ranges]
    else:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            chunks = list(ex.map(one, ranges))
    sums = []
    for c in chunks:
        sums.extend(c.tolist())
    return math.fsum(sums)


def nll_block_sums(spec, cols, block: int = BLOCK):
    n = len(next(iter(cols.values())))
    cache: dict = {}
    return block_sums(nll_terms(spec, cols, 0, n, 0, cache), block)


def sharded_nll(spec, cols, workers: int, block: int = BLOCK) -> float:
    """sharding.py:134-146 (partials exact, then one rounding)."""
    n = len(next(iter(cols.values())))
    b = shard_bounds(n, workers, block)
    cache: dict = {}
    sums = []
    for k in range(workers):
        size = b[k + 1] - b[k]
        if size == 0:
            continue
        sh = {name: c[b[k]:b[k + 1]] for name, c in cols.items()}
        sums.extend(block_sums(nll_terms(spec, sh, 0, size, b[k], cache), block).tolist())
    return math.fsum(sums)


# --- binned data (core.py:312-379, engine.py:246-276) ---------------------------------


def bin_width(lower: float, upper: float, n_bins: int) -> float:
    """core.py:334-336."""
    return (upper - lower) / n_bins


def bin_centers(axes):
    """core.py:345-362: axes = [(name, lower, upper, n_bins)], row-major grid."""
    grids = [np.array([lo + (b + 0.5) * (hi - lo) / nb for b in range(nb)]) for _, lo, hi, nb in axes]
    mesh = np.meshgrid(*grids, indexing="ij")
    return {a[0]: m.reshape(-1) for a, m in zip(axes, mesh)}


def bin_volume(axes) -> float:
    """core.py:338-342."""
    vol = 1.0
    for _, lo, hi, nb in axes:
        vol *= bin_width(lo, hi, nb)
    return vol


def fill(axes, cols, contents=None):
    """core.py:370-379: clip(int64(floor((x - lower) / width)), 0, nb - 1),
    row-major flat index, np.add.at of 1.0."""
    total_bins = int(np.prod([a[3] for a in axes]))
    contents = np.zeros(total_bins) if contents is None else contents
    n = len(cols[axes[0][0]])
    idx = np.zeros(n, dtype=np.int64)
    for name, lo, hi, nb in axes:
        k = np.floor((cols[name] - lo) / bin_width(lo, hi, nb)).astype(np.int64)
        np.clip(k, 0, nb - 1, out=k)
        idx = idx * nb + k
    np.add.at(contents, idx, 1.0)
    return contents


def binned_nll(spec, axes, contents) -> float:
    """engine.py:246-276: sum_b nu_b - n_b ln nu_b over the bin centres."""
    total = float(contents.sum())
    if total <= 0:
        raise OracleDensityError("EmptyDataSet")
    cache: dict = {}
    dens = spec_eval(spec, bin_centers(axes), cache) / spec_norm_cached(spec, cache)
    nu = total * dens * bin_volume(axes)
    observed = contents > 0
    bad = observed & ~(nu > 0.0)
    if bad.any():
        b = int(np.argmax(bad))
        raise OracleDensityError("NonPositiveExpectation", b, float(nu[b]))
    terms = nu.copy()
    terms[observed] -= contents[observed] * np.log(nu[observed])
    return math.fsum(terms.tolist())
