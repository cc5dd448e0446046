"""Binary SoA event ingest.

The reference reads events from CSV through Python lists (dataio.py:20-83,
core.py:259-282).  For 100M-event runs each observable is stored as one
little-endian float64 .npy column; :func:`load_npy` streams the rows a GPU
needs (its whole column, or its shard) straight from the files into HBM
(pfb_store_load_npy: pinned double buffer, reads overlapped with copies) and
runs the reference's strict range check on the device.  The dataset's host
columns are read-only memory maps of the same files: nothing is read on the
host unless a caller touches them, and the device copy is registered as their
HBM image so the NLL never uploads again.
"""

from __future__ import annotations

import ctypes
import os
from typing import Mapping, Sequence

import numpy as np

from . import _lib as L
from ._reference import errors as _E
from .datasets import DeviceDataSet

OutOfRange, ShapeMismatch = _E.OutOfRange, _E.ShapeMismatch


def save_npy(ds, directory: str) -> dict[str, str]:
    """Write each observable column of `ds` as <directory>/<name>.npy."""
    os.makedirs(directory, exist_ok=True)
    out = {}
    for name, col in ds.columns().items():
        path = os.path.join(directory, f"{name}.npy")
        np.save(path, np.ascontiguousarray(col, dtype="<f8"))
        out[name] = path
    return out


def npy_length(path: str) -> int:
    """Rows of a 1-D little-endian float64 .npy column (header only)."""
    n = ctypes.c_int64()
    code = L.lib().pfb_npy_length(os.fsencode(path), ctypes.byref(n))
    if code != L.OK:
        raise ShapeMismatch(f"{path!r} is not a 1-D '<f8' C-order .npy column")
    return n.value


def _paths_for(observables, paths) -> list[str]:
    if isinstance(paths, (str, os.PathLike)):
        return [os.path.join(os.fspath(paths), f"{o.name}.npy") for o in observables]
    if isinstance(paths, Mapping):
        return [os.fspath(paths[o.name]) for o in observables]
    paths = [os.fspath(p) for p in paths]
    if len(paths) != len(observables):
        raise ShapeMismatch("need one column file per observable")
    return paths


def load_npy(observables: Sequence, paths, begin: int = 0, end: int | None = None, device: int = 0,
             check: bool = True):
    """Rows [begin, end) of the observables' column files as an
    DeviceDataSet whose device copy is already in HBM."""
    from .engine import device_context
    from .mcgen import _device_store

    observables = list(observables)
    files = _paths_for(observables, paths)
    lengths = [npy_length(p) for p in files]
    if len(set(lengths)) != 1:
        raise ShapeMismatch(f"column files have unequal lengths {lengths}")
    total = lengths[0]
    end = total if end is None else int(end)
    begin = int(begin)
    if not 0 <= begin <= end <= total:
        raise ValueError(f"rows [{begin}, {end}) outside [0, {total})")
    n = end - begin
    if n == 0:
        return DeviceDataSet.from_columns(observables, [np.empty(0) for _ in files], device=None)
    ctx = device_context(device)
    st = _device_store(ctx, len(files), n)
    try:
        for c, path in enumerate(files):
            L.check(L.lib().pfb_store_load_npy(st, c, os.fsencode(path), begin, 0, n), "pfb_store_load_npy")
        if check:
            for c, obs in enumerate(observables):
                bad = ctypes.c_int64()
                val = ctypes.c_double()
                L.check(L.lib().pfb_store_check_range(st, c, 0, n, float(obs.lower), float(obs.upper),
                                                      ctypes.byref(bad), ctypes.byref(val)), "pfb_store_check_range")
                if bad.value >= 0:
                    raise OutOfRange(c, float(val.value), obs.name)
    except BaseException:
        L.lib().pfb_store_destroy(st)
        raise
    cols = [np.load(p, mmap_mode="r")[begin:end] for p in files]
    return DeviceDataSet.adopt_store(observables, cols, ctx, st)


def load_npy_shard(observables: Sequence, paths, rank: int, world: int, device: int = 0, check: bool = True):
    """This rank's shard (reference shard() bounds, sharding.py:80-85) of the
    column files -- each GPU reads only its own rows."""
    from .engine import shard_bounds

    files = _paths_for(list(observables), paths)
    b = shard_bounds(npy_length(files[0]), world)
    return load_npy(observables, files, b[rank], b[rank + 1], device=device, check=check)
