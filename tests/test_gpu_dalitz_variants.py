"""Dalitz structures beyond C3 against the reference (tests/golden/dalitz_variants.npz):
K = 2 and 3 (compile-time K, generic structure), a K pi pi channel with unequal
daughter masses (non-zero Zemach constants on every pair), and K = 5 (the
any-K evaluator) -- through the product kernels (pipeline 1) and the SIMT
reference-tree kernel (pipeline 0)."""

import os

import numpy as np
import pytest

from tests import models
from paper_1710_08826_b200._reference import parafit as P

pytestmark = pytest.mark.gpu

RTOL = 1e-10


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


@pytest.mark.parametrize("pipeline", [1, 0])
@pytest.mark.parametrize("name", sorted(models.DALITZ_VARIANTS))
def test_dalitz_variant_matches_reference(pf, golden_dir, name, pipeline):
    from paper_1710_08826_b200 import _lib as L

    g = np.load(os.path.join(golden_dir, "dalitz_variants.npz"))
    (s12, s13), pdf, terms = models.dalitz_variant(P, name)
    ds = models.dataset([s12, s13], [g[f"{name}__s12"], g[f"{name}__s13"]])
    ctx = pf.device_context(0)
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, pipeline), "pfb_ctx_set_pipeline")
    try:
        got = [pf.nll(pdf, ds)]
        P.set_value(terms[1].magnitude, terms[1].magnitude.value * 1.1)
        P.set_value(terms[-1].phase, terms[-1].phase.value + 0.2)
        got.append(pf.nll(pdf, ds))
    finally:
        L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, 1), "pfb_ctx_set_pipeline")
    for a, b in zip(got, g[f"{name}__nll"]):
        assert abs(a - b) <= RTOL * abs(b), (name, a, b)
