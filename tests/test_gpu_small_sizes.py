"""Tail handling of every shell at small and ragged sizes: 1, 2, 3, 17, 4095,
4096, 4097, 8193 and 12289 events (odd last events, lone tail blocks, a tail
after full blocks) for the C1 SumPdf, C2 ProdPdf, C3 Dalitz, C2p gaussian x
polynomial and a lone-polynomial model, through pipelines 1 / 2 / 3 (bulk,
TMA-unit and per-warp staging kernels) and 0 (SIMT) -- each NLL within 1e-10
of the reference's own nll on the same events (P/engine.py:214-243), and the
shells of a product evaluator (staging kernels and the SIMT kernel at 1 / 2 /
4 / 8 warps per block) bitwise equal to each other."""

import os

import numpy as np
import pytest

from paper_1710_08826_b200._reference import parafit as P
from tests import models

pytestmark = pytest.mark.gpu

SIZES = (1, 2, 3, 17, 4095, 4096, 4097, 8193, 12289)


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def model(name):
    if name == "c1":
        x, pdf, _ = models.c1()
        return [x], pdf
    if name == "c2":
        obs, pdf, _ = models.c2()
        return list(obs), pdf
    if name == "c3":
        obs, pdf, _ = models.c3(grid=(128, 128))
        return list(obs), pdf
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", 0.0, 10.0)
    poly = P.polynomial(y if name == "c2p" else x,
                        [P.Variable(f"q{k}", v, -10.0, 10.0) for k, v in enumerate((1.0, 0.3, 0.05))])
    if name == "poly":
        return [x], poly
    return [x, y], P.prod_pdf([P.gaussian(x, P.Variable("m", 5.0, 0.0, 10.0), P.Variable("s", 1.0, 0.1, 5.0)),
                               poly])


def events(obs, n, rng):
    if len(obs) == 2 and obs[0].name == "s12":
        g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c3_dalitz.npz"))
        return [g["s12"][:n], g["s13"][:n]]
    return [np.clip(rng.normal(5.0, 1.5, n), o.lower, o.upper) for o in obs]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c2p", "poly"])
def test_small_and_ragged_sizes_every_shell(pf, name):
    rng = np.random.default_rng(29)
    obs, pdf = model(name)
    ctx = pf.device_context(0)
    for n in SIZES:
        cols = events(obs, n, rng)
        if len(cols[0]) < n:
            continue
        ds = pf.DeviceDataSet.from_columns(obs, cols, device=None)
        snap = P.snapshot(pdf.param_closure())
        with pf.reference_norms():
            want = P.nll(pdf, ds, snap, P.Backend("serial"), P.NormalizationStore())
        got = {}
        try:
            for mode in (1, 2, 3, 0):
                ctx.set_pipeline(mode)
                got[mode] = pf.nll(pdf, ds)
        finally:
            ctx.set_pipeline(1)
        for mode, v in got.items():
            assert abs(v - want) <= 1e-10 * abs(want), (name, n, mode, v, want)
        if name in ("c1", "c3", "c2p", "poly"):  # product evaluators: every shell agrees bitwise
            assert got[1] == got[2] == got[3], (name, n, got)
            try:
                for w in (1, 2, 4, 8):  # the register-window SIMT kernel, P warps per block
                    ctx.set_warps_per_block(w)
                    assert pf.nll(pdf, ds) == got[1], (name, n, w)
            finally:
                ctx.set_warps_per_block(0)
