"""Device-resident event stores behind the reference's dataset classes.

:class:`DeviceDataSet` IS a reference ``UnbinnedDataSet`` (P/core.py:215-309):
the reference ``nll``/``FitManager``/``shard`` accept it unchanged.  The
reference keeps rows in Python lists (P/core.py:233) -- ~54 B per value and
seconds per 10M rows -- and materialises float64 columns on demand
(P/core.py:293-296).  A DeviceDataSet instead holds whole float64 columns
(SoA, north_star item 1) whose HBM copy is registered with the device
context, so the NLL never re-uploads them: columns produced on the GPU
(:mod:`.mcgen`, :mod:`.dataio`) are adopted as they are.  Row-wise appends
(``add_event``/``extend``) first hand the columns back to the reference
representation and then run the reference's own code.

:func:`bin_fill` and :func:`binned_nll` are the device versions of
``BinnedDataSet.fill`` (P/core.py:370-379) and ``binned_nll``
(P/engine.py:246-276) for the reference ``BinnedDataSet``.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _lib as L
from ._reference import core as ref_core
from ._reference import engine as ref_engine
from ._reference import errors as ref_errors


class DeviceDataSet(ref_core.UnbinnedDataSet):
    """Column-major events with an HBM copy; a reference ``UnbinnedDataSet``."""

    def __init__(self, observables: Sequence, lenient: bool = False):
        super().__init__(observables, lenient)
        self._cols: list[np.ndarray] | None = None

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_columns(cls, observables: Sequence, columns: Sequence[np.ndarray], device: int | None = 0,
                     check: bool = True) -> "DeviceDataSet":
        """Adopt whole float64 columns (no copy when already contiguous float64).

        With ``check`` the reference's strict range check (P/core.py:262-272:
        first row with x < lower, x > upper or non-finite -> OutOfRange) runs
        on the device copy; ``device=None`` skips the upload (host columns
        only, uploaded on the first NLL)."""
        ds = cls(observables)
        cols = [c if (isinstance(c, np.ndarray) and c.dtype == np.float64 and c.ndim == 1 and c.flags.c_contiguous)
                else np.ascontiguousarray(c, dtype=np.float64).reshape(-1) for c in columns]
        if len(cols) != len(ds.observables) or any(len(c) != len(cols[0]) for c in cols):
            raise ref_errors.ShapeMismatch("columns do not match the observables")
        if device is not None and len(cols[0]):
            from .engine import device_context

            st = device_context(device).store_for(cols)
            if check:
                check_range(st, ds.observables, len(cols[0]))
        elif check:
            for i, (obs, c) in enumerate(zip(ds.observables, cols)):
                bad = (c < obs.lower) | (c > obs.upper) | ~np.isfinite(c)
                if bad.any():
                    j = int(np.argmax(bad))
                    raise ref_errors.OutOfRange(i, float(c[j]), obs.name)
        ds._cols = cols
        return ds

    @classmethod
    def adopt_store(cls, observables: Sequence, columns: Sequence[np.ndarray], ctx=None, store=None) -> "DeviceDataSet":
        """Columns whose HBM copy already exists (and whose range check already
        ran on it): with `store`, register the pair in `ctx`; without, the pair
        is already registered.  No upload."""
        ds = cls(observables)
        ds._cols = list(columns)
        if store is not None and len(ds._cols[0]):
            ctx.adopt(ds._cols, store)
        return ds

    # -- the reference interface ------------------------------------------------
    @property
    def n_events(self) -> int:
        if self._cols is not None:
            return len(self._cols[0])
        return super().n_events

    def _materialize(self) -> list[np.ndarray]:
        if self._cols is not None:
            return self._cols
        return super()._materialize()

    def _to_rows(self) -> None:
        """Hand the columns to the reference's list storage before a row append."""
        if self._cols is not None:
            self._lists = [c.tolist() for c in self._cols]
            self._cols = None
            self._arrays = None

    def add_event(self, row) -> None:
        self._to_rows()
        super().add_event(row)

    def extend(self, columns) -> None:
        self._to_rows()
        super().extend(columns)


def check_range(store, observables, n: int) -> None:
    """The reference dataset range check (P/core.py:262-272) on a device store."""
    for c, obs in enumerate(observables):
        bad = ctypes.c_int64()
        val = ctypes.c_double()
        L.check(L.lib().pfb_store_check_range(store, c, 0, n, float(obs.lower), float(obs.upper),
                                              ctypes.byref(bad), ctypes.byref(val)), "pfb_store_check_range")
        if bad.value >= 0:
            raise ref_errors.OutOfRange(c, float(val.value), obs.name)


def as_device_dataset(ds, device: int = 0) -> DeviceDataSet:
    """A DeviceDataSet over the same columns as a reference dataset."""
    if isinstance(ds, DeviceDataSet):
        return ds
    cols = ds.columns()
    return DeviceDataSet.from_columns(ds.observables, [cols[o.name] for o in ds.observables], device=device,
                                      check=False)


# --- binned data ------------------------------------------------------


def bin_fill(binned, ds, device: int = 0) -> None:
    """``BinnedDataSet.fill`` (P/core.py:370-379) on the GPU (pfb_bin_fill): per
    axis clip(int64(floor((x - lower) / width)), 0, n_bins - 1), row-major
    flat index, counts added per bin -- bit-exact with the reference."""
    from .engine import device_context

    cols = [ds.column(obs.name) for obs in binned.observables]
    if ds.n_events == 0:
        return
    ctx = device_context(device)
    st = ctx.store_for(cols)
    naxes = len(binned.observables)
    idx = np.arange(naxes, dtype=np.int32)
    lower = np.array([o.lower for o in binned.observables], dtype=np.float64)
    width = np.array([binned.bin_width(a) for a in range(naxes)], dtype=np.float64)
    nbins = np.array(binned.n_bins, dtype=np.int64)
    contents = binned.contents
    if not (contents.dtype == np.float64 and contents.flags.c_contiguous):
        raise ref_errors.ShapeMismatch("BinnedDataSet.contents must be contiguous float64")
    L.check(L.lib().pfb_bin_fill(ctx.handle, st, 0, ds.n_events, naxes, L.dptr(idx), L.dptr(lower),
                                 L.dptr(width), L.dptr(nbins), L.dptr(contents)), "pfb_bin_fill")


_centers_cache: dict[int, tuple] = {}


def _device_centers(binned):
    """``centers()`` computed once per binning (immutable), so the same arrays
    -- and their HBM copy -- serve every call."""
    hit = _centers_cache.get(id(binned))
    if hit is None or hit[0] is not binned:
        hit = (binned, {k: np.ascontiguousarray(v) for k, v in binned.centers().items()})
        _centers_cache[id(binned)] = hit
    return hit[1]


def binned_nll(pdf, ds, snap=None, backend=None, store=None) -> float:
    """Poisson NLL over bins, sum_b [nu_b - n_b ln nu_b] (P/engine.py:246-276):
    densities at the bin centres and the exact sum on the GPU
    (pfb_binned_nll); nu_b = total * p_b * bin volume as the reference."""
    from .engine import DeviceBackend, device_context, raise_for

    total = ds.total
    if total <= 0:
        raise ref_errors.EmptyDataSet("binned dataset has no content")
    store = store if store is not None else ref_engine.NormalizationStore()
    if snap is None:
        snap = ref_core.snapshot(pdf.param_closure())
    norms = ref_engine.resolve_norms(pdf, snap, store)
    device = backend.devices[0] if isinstance(backend, DeviceBackend) else 0
    ctx = device_context(device)
    centers = _device_centers(ds)
    needed = sorted({name for node in pdf.walk() for name in node.observable_names()})
    missing = set(needed) - set(centers)
    if missing:
        raise KeyError(f"binned dataset lacks observables {sorted(missing)}")
    arrays = [centers[name] for name in needed]
    plan = ctx.plan_for(pdf, tuple(needed))
    st = ctx.store_for(arrays)
    vals, nv = plan.pack(snap, norms)
    contents = np.ascontiguousarray(ds.contents, dtype=np.float64)
    out = ctypes.c_double()
    err = L.PfbErr()
    code = L.lib().pfb_binned_nll(ctx.handle, plan.handle, st, L.dptr(contents), contents.size, float(total),
                                  float(ds.bin_volume()), L.dptr(vals), len(vals), L.dptr(nv), len(nv),
                                  ctypes.byref(out), ctypes.byref(err))
    raise_for(err, code, "pfb_binned_nll")
    return out.value
