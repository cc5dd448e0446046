"""Three-body Dalitz model: host description + GPU normalisation integrals.

Model description mirrors the reference (dalitz.py:47-117, 355-377):
DecayChannel, ResonanceTerm, dalitz_pdf with parameters ordered
[mass, width, magnitude, phase] per term.  Per-event intensities are
evaluated only on the device (pfb_nll).  The normalisation

    norm = sum_ij c_i conj(c_j) I_ij,   I_ij = sum_grid A_i conj(A_j) dA

keeps the reference's structure (dalitz.py:282-349): the midpoint grid, its
bit-exact kinematic mask and the stale-row overlap integrals are computed on
the GPU by a pfb_grid (one per Dalitz node), only for terms whose shape
fingerprint (pair, spin, mass, width) moved; the K x K contraction with the
coefficients stays a host scalar, as in the reference.

The small numpy helpers (s13_limits, in_boundary_mask) exist for synthetic
event generation and tests; they are not on the NLL path.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as L
from . import engine as _engine
from .core import Variable
from .errors import DegenerateGrid, NonPositiveNorm
from .pdf import PdfNode, pval, register_norm

PAIRS = (12, 13, 23)
DEFAULT_GRID = (400, 400)


@dataclass(frozen=True)
class DecayChannel:
    mother_mass: float
    m1: float
    m2: float
    m3: float

    def __post_init__(self):
        daughters = self.m1 + self.m2 + self.m3
        if not (self.mother_mass > daughters >= 0.0):
            raise ValueError(f"need mother mass {self.mother_mass} > sum of daughters {daughters} >= 0")

    @property
    def mass_sum_sq(self) -> float:
        return self.mother_mass**2 + self.m1**2 + self.m2**2 + self.m3**2

    @property
    def s12_range(self) -> tuple[float, float]:
        return ((self.m1 + self.m2) ** 2, (self.mother_mass - self.m3) ** 2)

    @property
    def s13_range(self) -> tuple[float, float]:
        return ((self.m1 + self.m3) ** 2, (self.mother_mass - self.m2) ** 2)

    def s23(self, s12, s13):
        return self.mass_sum_sq - s12 - s13


@dataclass
class ResonanceTerm:
    pair: int
    mass: Variable
    width: Variable
    spin: int
    magnitude: Variable
    phase: Variable
    name: str = ""

    def __post_init__(self):
        if self.pair not in PAIRS:
            raise ValueError(f"pair must be one of {PAIRS}, got {self.pair}")
        if self.spin not in (0, 1):
            raise ValueError(f"spin must be 0 or 1, got {self.spin}")
        if not self.mass.value > 0:
            raise ValueError("resonance mass must be > 0")
        if not self.width.value > 0:
            raise ValueError("resonance width must be > 0")

    def shape_fingerprint(self) -> tuple:
        return (self.pair, self.spin, self.mass.value, self.mass.generation, self.width.value,
                self.width.generation)


# --- host helpers for generation / tests (not on the NLL path) ----------------------


def s13_limits(s12, ch: DecayChannel):
    s12 = np.asarray(s12, dtype=np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        rs = np.sqrt(s12)
        e1 = (s12 + ch.m1**2 - ch.m2**2) / (2.0 * rs)
        e3 = (ch.mother_mass**2 - s12 - ch.m3**2) / (2.0 * rs)
        p1 = np.sqrt(e1 * e1 - ch.m1**2)
        p3 = np.sqrt(e3 * e3 - ch.m3**2)
        esum = (e1 + e3) ** 2
        return esum - (p1 + p3) ** 2, esum - (p1 - p3) ** 2


def in_boundary_mask(s12, s13, ch: DecayChannel) -> np.ndarray:
    s12 = np.asarray(s12, dtype=np.float64)
    s13 = np.asarray(s13, dtype=np.float64)
    lo12, hi12 = ch.s12_range
    lo, hi = s13_limits(s12, ch)
    with np.errstate(invalid="ignore"):
        return (s12 >= lo12) & (s12 <= hi12) & (s13 >= lo) & (s13 <= hi)


def coefficients(terms: Sequence[ResonanceTerm], snap=None) -> np.ndarray:
    mags = np.array([pval(t.magnitude, snap) for t in terms], dtype=np.float64)
    phases = np.array([pval(t.phase, snap) for t in terms], dtype=np.float64)
    return mags * np.exp(1j * phases)


# --- device grid -----------------------------------------------------------------------


def _desc(ch: DecayChannel, terms=()) -> L.PfbDalitzDesc:
    d = L.PfbDalitzDesc()
    d.mother_mass, d.m1, d.m2, d.m3 = ch.mother_mass, ch.m1, ch.m2, ch.m3
    d.nterms = len(terms)
    for k, t in enumerate(terms):
        d.pair[k] = int(t.pair)
        d.spin[k] = int(t.spin)
    return d


class DeviceGrid:
    """A pfb_grid: midpoint nodes, bit-exact mask and per-term amplitude rows
    resident in HBM.  ``row_fp[k]`` is the shape fingerprint row k was last
    computed for, so a row is reused only if it really holds that shape."""

    def __init__(self, ctx, ch: DecayChannel, grid: tuple[int, int]):
        nx, ny = grid
        if nx < 32 or ny < 32:
            raise DegenerateGrid(f"need >= 32 nodes per axis, got {grid}")
        self.ctx = ctx
        self.grid = (int(nx), int(ny))
        self._desc = _desc(ch)
        h = ctypes.c_void_p()
        L.check(L.lib().pfb_grid_create(ctx.handle, ctypes.byref(self._desc), nx, ny, ctypes.byref(h)),
                "pfb_grid_create")
        self.handle = h
        n = ctypes.c_int64()
        area = ctypes.c_double()
        L.check(L.lib().pfb_grid_info(h, ctypes.byref(n), ctypes.byref(area)), "pfb_grid_info")
        self.n_inside = n.value
        self.area = area.value
        self.row_fp: dict[int, tuple] = {}

    def mask(self) -> np.ndarray:
        out = np.empty(self.grid[0] * self.grid[1], dtype=np.uint8)
        L.check(L.lib().pfb_grid_mask(self.handle, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))),
                "pfb_grid_mask")
        return out.astype(bool)

    def integrals(self, terms, shapes, fps, stale, matrix: np.ndarray) -> np.ndarray:
        K = len(terms)
        # a stale entry (i, j) needs rows i and j on the device; with any term
        # stale every row takes part, so refresh the rows not holding their shape
        any_stale = any(stale)
        rows = np.array([1 if any_stale and self.row_fp.get(k) != fps[k] else 0 for k in range(K)],
                        dtype=np.uint8)
        pair = np.array([t.pair for t in terms], dtype=np.int32)
        spin = np.array([t.spin for t in terms], dtype=np.int32)
        mw = np.array(shapes, dtype=np.float64).reshape(-1)
        st = np.array(stale, dtype=np.uint8)
        buf = np.ascontiguousarray(np.stack([matrix.real, matrix.imag], axis=-1).reshape(-1), dtype=np.float64)
        L.check(L.lib().pfb_grid_integrals(
            self.ctx.handle, self.handle, K,
            pair.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            spin.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            L.dptr(mw), rows.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
            st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), L.dptr(buf)), "pfb_grid_integrals")
        for k in range(K):
            if rows[k]:
                self.row_fp[k] = fps[k]
        out = buf.reshape(K, K, 2)
        return out[..., 0] + 1j * out[..., 1]

    def close(self) -> None:
        if self.handle:
            L.lib().pfb_grid_destroy(self.handle)
            self.handle = None


def device_grid(ch: DecayChannel, grid, owner=None, ctx=None) -> DeviceGrid:
    ctx = ctx or _engine.device_context(0)
    key = (owner, ch, tuple(grid))
    g = ctx.grids.get(key)
    if g is None:
        g = DeviceGrid(ctx, ch, tuple(grid))
        ctx.grids[key] = g
    return g


def integration_grid(ch: DecayChannel, grid: tuple[int, int] = DEFAULT_GRID):
    """Flattened node centres, the device-computed in-boundary mask and cell area
    (reference dalitz.py:246-264)."""
    nx, ny = grid
    if nx < 32 or ny < 32:
        raise DegenerateGrid(f"need >= 32 nodes per axis, got {grid}")
    (lo12, hi12), (lo13, hi13) = ch.s12_range, ch.s13_range
    dx = (hi12 - lo12) / nx
    dy = (hi13 - lo13) / ny
    g12, g13 = np.meshgrid(lo12 + (np.arange(nx) + 0.5) * dx, lo13 + (np.arange(ny) + 0.5) * dy, indexing="ij")
    g = device_grid(ch, grid)
    return g12.reshape(-1), g13.reshape(-1), g.mask(), dx * dy


@dataclass
class IntegralCache:
    """Hermitian overlap matrix with per-term fingerprints (reference dalitz.py:267-279)."""

    matrix: np.ndarray
    fingerprints: tuple
    grid: tuple
    amplitudes: object = field(repr=False, default=None)  # the DeviceGrid holding the rows

    def __post_init__(self):
        n = len(self.fingerprints)
        if self.matrix.shape != (n, n):
            raise ValueError("integral matrix size does not match term count")


def compute_integrals(terms: Sequence[ResonanceTerm], ch: DecayChannel, grid=DEFAULT_GRID,
                      prior: IntegralCache | None = None, snap=None, owner=None) -> IntegralCache:
    """Overlap integrals with prior reuse (reference dalitz.py:282-329), on the GPU."""
    fps = tuple(t.shape_fingerprint() for t in terms)
    grid = tuple(grid)
    if prior is not None and prior.grid == grid and prior.fingerprints == fps:
        return prior
    dg = device_grid(ch, grid, owner=owner if owner is not None else tuple(id(t) for t in terms))
    n = len(terms)
    stale = [
        prior is None or prior.grid != grid or i >= len(prior.fingerprints)
        or prior.fingerprints[i] != fps[i] or prior.amplitudes is None
        for i in range(n)
    ]
    matrix = np.zeros((n, n), dtype=np.complex128)
    if prior is not None and not all(stale):
        m = min(n, prior.matrix.shape[0])
        matrix[:m, :m] = prior.matrix[:m, :m]
    shapes = [(pval(t.mass, snap), pval(t.width, snap)) for t in terms]
    matrix = dg.integrals(terms, shapes, fps, stale, matrix)
    return IntegralCache(matrix=matrix, fingerprints=fps, grid=grid, amplitudes=dg)


def dalitz_norm(terms: Sequence[ResonanceTerm], cache: IntegralCache, snap=None) -> float:
    """sum_ij c_i conj(c_j) I_ij (reference dalitz.py:332-349)."""
    if len(terms) != len(cache.fingerprints):
        raise ValueError("integral cache does not match the term list")
    c = coefficients(terms, snap)
    total = complex(np.dot(c, cache.matrix @ np.conj(c)))
    scale = max(abs(total.real), 1e-300)
    if abs(total.imag) > 1e-10 * scale:
        raise NonPositiveNorm(f"overlap sum has a non-negligible imaginary part: {total!r}")
    if not total.real > 0.0:
        raise NonPositiveNorm(f"overlap sum {total.real!r} is not positive")
    return total.real


def dalitz_pdf(terms: Sequence[ResonanceTerm], ch: DecayChannel, s12_obs: Variable | None = None,
               s13_obs: Variable | None = None, grid=DEFAULT_GRID) -> PdfNode:
    if not terms:
        raise ValueError("need at least one resonance term")
    if s12_obs is None:
        s12_obs = Variable.observable("s12", *ch.s12_range)
    if s13_obs is None:
        s13_obs = Variable.observable("s13", *ch.s13_range)
    params: list[Variable] = []
    for t in terms:
        params.extend((t.mass, t.width, t.magnitude, t.phase))
    return PdfNode("dalitz", [s12_obs, s13_obs], params, payload=(tuple(terms), ch, tuple(grid)))


def _dalitz_norm_pure(node, snap, child_norms):
    terms, ch, grid = node.payload
    cache = compute_integrals(terms, ch, grid, prior=None, snap=snap, owner=("pure", node.id))
    return dalitz_norm(terms, cache, snap)


def dalitz_cached_norm(node, snap, store):
    """Norm hook (reference dalitz.py:393-410) with GPU integrals."""
    terms, ch, grid = node.payload
    key = ("dalitz-integrals", node.id)
    entry = store.get(key)
    prior = entry[1] if entry is not None else None
    cache = compute_integrals(terms, ch, grid, prior=prior, snap=snap, owner=node.id)
    if cache is not prior:
        if prior is None or prior.grid != cache.grid:
            changed = len(cache.fingerprints)
        else:
            changed = sum(1 for i, fp in enumerate(cache.fingerprints)
                          if i >= len(prior.fingerprints) or prior.fingerprints[i] != fp)
        store.kernel_evals += changed
        store.put(key, cache.fingerprints, cache)
    return dalitz_norm(terms, cache, snap)


register_norm("dalitz", _dalitz_norm_pure)
_engine.register_cached_norm("dalitz", dalitz_cached_norm)
