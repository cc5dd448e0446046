"""Dalitz normalisation on the GPU for the reference's ``dalitz_pdf`` nodes.

The model (``DecayChannel``, ``ResonanceTerm``, ``dalitz_pdf``) is the
reference's (P/dalitz.py:47-117,355-377).  The per-event coherent sum runs in
the fused NLL kernel; this module moves the normalisation integrals
(P/dalitz.py:246-349) to HBM:

* :class:`DeviceGrid` -- the midpoint grid, its **bit-exact** kinematic mask
  (P/dalitz.py:127-150,246-264) and one amplitude row per term, resident in
  HBM (pfb_grid_*);
* :func:`compute_integrals` -- the reference's reuse rules (P/dalitz.py:282-329):
  nothing recomputed when every term's shape fingerprint (pair, spin, mass,
  width) is unchanged; otherwise only stale rows are re-evaluated and only
  pairs touching a stale term re-integrated, on the device, with the exact
  accumulator.  Returns the reference's own ``IntegralCache``;
* :func:`dalitz_cached_norm` -- the ``register_cached_norm("dalitz", ...)``
  hook (P/dalitz.py:393-410 semantics: store key ``("dalitz-integrals",
  node.id)``, ``kernel_evals`` += number of changed terms), finishing with the
  reference's own ``dalitz_norm`` (P/dalitz.py:332-349) for the K x K
  contraction with the coefficients.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from ._reference import dalitz as ref_dalitz
from ._reference import errors as ref_errors
from ._reference import pdf as ref_pdf


def _desc(ch, terms=()) -> L.PfbDalitzDesc:
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

    def __init__(self, ctx, ch, grid: tuple[int, int]):
        nx, ny = grid
        if nx < 32 or ny < 32:
            raise ref_errors.DegenerateGrid(f"need >= 32 nodes per axis, got {grid}")
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
        """The in-boundary mask over the nx*ny row-major nodes (device-computed)."""
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


def device_grid(ch, grid, owner=None, ctx=None) -> DeviceGrid:
    from .engine import device_context

    ctx = ctx or device_context(0)
    key = (owner, ch, tuple(grid))
    g = ctx.grids.get(key)
    if g is None:
        g = DeviceGrid(ctx, ch, tuple(grid))
        ctx.grids[key] = g
    return g


def grid_mask(ch, grid=ref_dalitz.DEFAULT_GRID, ctx=None) -> np.ndarray:
    """The device-computed in-boundary mask of ``integration_grid`` (P/dalitz.py:246-264)."""
    return device_grid(ch, grid, owner="mask", ctx=ctx).mask()


def compute_integrals(terms, ch, grid=ref_dalitz.DEFAULT_GRID, prior=None, snap=None, owner=None, ctx=None):
    """Overlap integrals with the reference's prior-reuse rules
    (P/dalitz.py:282-329), evaluated on the GPU.  Returns a reference
    ``IntegralCache`` whose ``amplitudes`` is the :class:`DeviceGrid` holding
    the rows in HBM."""
    fps = tuple(t.shape_fingerprint() for t in terms)
    grid = tuple(grid)
    if prior is not None and prior.grid == grid and prior.fingerprints == fps:
        return prior
    dg = device_grid(ch, grid, owner=owner if owner is not None else tuple(id(t) for t in terms), ctx=ctx)
    n = len(terms)
    on_device = prior is not None and isinstance(prior.amplitudes, DeviceGrid)
    stale = [
        not on_device or prior.grid != grid or i >= len(prior.fingerprints) or prior.fingerprints[i] != fps[i]
        for i in range(n)
    ]
    matrix = np.zeros((n, n), dtype=np.complex128)
    if on_device and not all(stale):
        m = min(n, prior.matrix.shape[0])
        matrix[:m, :m] = prior.matrix[:m, :m]
    shapes = [(ref_pdf._pval(t.mass, snap), ref_pdf._pval(t.width, snap)) for t in terms]
    matrix = dg.integrals(terms, shapes, fps, stale, matrix)
    return ref_dalitz.IntegralCache(matrix=matrix, fingerprints=fps, grid=grid, amplitudes=dg)


def dalitz_cached_norm(node, snap, store):
    """``register_cached_norm("dalitz", ...)`` hook with GPU integrals
    (P/dalitz.py:393-410 semantics)."""
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
    return ref_dalitz.dalitz_norm(terms, cache, snap)
