"""Generic PDF trees on the device against the reference (tests/golden/trees.npz):
polynomial leaves with Gauss-Legendre norms, nested add/prod, three-term
sums, three observables, single leaves -- through every kernel family
(pipeline 1: unit-sum / product kernels, 2: reference-tree TMA, 0: SIMT)."""

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


@pytest.mark.parametrize("pipeline", [1, 2, 0, 3])
@pytest.mark.parametrize("name", [t[0] for t in models.TREES])
def test_tree_nll_matches_reference(pf, golden_dir, name, pipeline):
    from paper_1710_08826_b200 import _lib as L

    g = np.load(os.path.join(golden_dir, "trees.npz"))
    spec = dict(models.TREES)[name]
    ctx = pf.device_context(0)
    L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, pipeline), "pfb_ctx_set_pipeline")
    try:
        for scale, want in zip((0.0, 0.01, -0.02), g[f"{name}__nll"]):
            root, obs, _ = models.build_tree(P, models.perturb(spec, scale))
            names = sorted(obs)
            ds = models.dataset([obs[c] for c in names], [g[f"{name}__{c}"] for c in names])
            got = pf.nll(root, ds)
            assert abs(got - want) <= RTOL * abs(want), (name, scale, got, want)
    finally:
        L.check(L.lib().pfb_ctx_set_pipeline(ctx.handle, 1), "pfb_ctx_set_pipeline")
