"""Binary SoA ingest straight to HBM: a dataset loaded from
column files gives the in-memory dataset's NLL bit for bit, shards load only
their rows, and the reference's range check raises the same OutOfRange."""

import os

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def test_load_equals_in_memory_and_shards(pf, golden_dir, tmp_path):
    from paper_1710_08826_b200 import dataio
    from paper_1710_08826_b200.sharding import shard_bounds

    g = np.load(os.path.join(golden_dir, "c2_prod.npz"))
    (x, y), pdf, params = models.c2()
    mem = models.dataset([x, y], [g["x"], g["y"]])
    files = dataio.save_npy(mem, str(tmp_path))
    ds = dataio.load_npy([x, y], str(tmp_path))
    assert ds.n_events == mem.n_events
    assert pf.nll(pdf, ds) == pf.nll(pdf, mem)
    assert np.array_equal(np.asarray(ds.column("x")), g["x"])
    # each rank's shard: its rows only, and the exact partials recombine
    from paper_1710_08826_b200 import sharding

    w = 3
    b = shard_bounds(mem.n_events, w)
    parts = []
    for r in range(w):
        sh = dataio.load_npy_shard([x, y], files, r, w)
        assert sh.n_events == b[r + 1] - b[r]
        assert np.array_equal(np.asarray(sh.column("y")), g["y"][b[r]:b[r + 1]])
        snap = P.snapshot(pdf.param_closure())
        norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
        parts.append(pf.nll_block_sums(pdf, sh.columns(), snap, norms, 0, sh.n_events))
    total = sharding.round_acc(sharding.acc_of_values(np.concatenate(parts)))
    assert total == pf.nll(pdf, mem)


def test_range_check_matches_reference_error(pf, tmp_path):
    from paper_1710_08826_b200 import dataio
    from paper_1710_08826_b200._reference import errors as E

    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    xs = np.linspace(0.0, 10.0, 50001)
    ys = np.full_like(xs, 5.0)
    ys[31337] = 10.5
    ys[40000] = np.nan
    np.save(tmp_path / "x.npy", xs)
    np.save(tmp_path / "y.npy", ys)
    with pytest.raises(E.OutOfRange) as ei:
        dataio.load_npy([x, y], str(tmp_path))
    want = None
    try:
        models.dataset([x, y], [xs, ys])
    except E.OutOfRange as exc:
        want = exc
    assert want is not None and (ei.value.index, ei.value.value, ei.value.name) == (want.index, want.value, want.name)


def test_store_round_trip_pageable_and_pinned(pf):
    """pfb_store_upload / pfb_store_download move columns bit for bit: the
    multi-lane pinned-staged download into pageable memory (sizes that split
    unevenly over the lanes and staging chunks) and the direct copy into
    pinned memory."""
    import ctypes

    import numpy as np
    import torch

    from paper_1710_08826_b200 import _lib as L

    ctx = pf.device_context(0)
    rng = np.random.default_rng(7)
    for n in (3, 1_048_577, 5_000_003):
        src = rng.normal(size=n)
        st = ctypes.c_void_p()
        L.check(L.lib().pfb_store_create(ctx.handle, 1, n, ctypes.byref(st)), "pfb_store_create")
        try:
            L.check(L.lib().pfb_store_upload(st, 0, L.dptr(src), 0, n), "pfb_store_upload")
            out = np.empty(n)
            L.check(L.lib().pfb_store_download(st, 0, L.dptr(out), 0, n), "pfb_store_download")
            assert out.tobytes() == src.tobytes()
            pinned = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
            L.check(L.lib().pfb_store_download(st, 0, L.dptr(pinned), 0, n), "pfb_store_download")
            assert pinned.tobytes() == src.tobytes()
            part = np.empty(n - 1)
            L.check(L.lib().pfb_store_download(st, 0, L.dptr(part), 1, n - 1), "pfb_store_download")
            assert part.tobytes() == src[1:].tobytes()
        finally:
            L.lib().pfb_store_destroy(st)
