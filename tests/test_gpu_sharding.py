"""Device partials behind the reference's shard / reduce (P/sharding.py:68-146)
and error propagation on every multi-part path.

* ``partial_nll`` returns the reference ``PartialSum`` whose components are
  an exact expansion of the device accumulator: the reference
  ``reduce_partials`` merges them bitwise into the single-GPU NLL, and mixes
  them with the reference's own host partials.
* ``FractionOutOfRange`` (P/pdf.py:205-210) is raised -- never a finite NLL --
  on the multi-device in-process split, device ``sharded_nll`` and the fused
  one-process-per-GPU path, even where the densities stay positive.
"""

import math

import numpy as np
import pytest

from paper_1710_08826_b200._reference import errors as E
from paper_1710_08826_b200._reference import parafit as P
from tests import models

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    if L.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device")
    return pf


def _c2(n, seed=3):
    rng = np.random.default_rng(seed)
    (x, y), pdf, params = models.c2()
    ds = models.dataset([x, y], [np.clip(rng.normal(5, 1, n), 0, 10), np.clip(rng.exponential(2.5, n), 0, 10)])
    return pdf, ds, params


@pytest.mark.parametrize("workers", [1, 2, 3, 8])
def test_device_partials_reduce_bitwise_through_the_reference(pf, workers):
    pdf, ds, _ = _c2(40 * 4096 + 321)
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    whole = pf.nll(pdf, ds, snap)
    parts = [pf.partial_nll(sh, pdf, snap, norms) for sh in P.shard(ds, workers)]
    assert all(isinstance(p, P.PartialSum) and p.components for p in parts)
    assert P.reduce_partials(parts) == whole  # block-aligned shards: the single-GPU bits
    assert pf.sharded_nll(pdf, ds, snap, workers=workers) == whole
    with pf.reference_norms():
        ref_parts = [P.partial_nll(sh, pdf, snap, norms) for sh in P.shard(ds, workers)]
        ref_whole = P.sharded_nll(pdf, ds, snap, workers=workers)
    assert abs(P.reduce_partials(ref_parts) - whole) <= 1e-10 * abs(whole)
    # device and host partials merge in one reduction
    mixed = [parts[0]] + ref_parts[1:]
    assert abs(P.reduce_partials(mixed) - ref_whole) <= 1e-10 * abs(ref_whole)


def test_partial_error_carries_global_index(pf):
    # reference tests/test_sharding.py:114-129 (global index 1500 in shard 1 of 2... here 9000)
    x = P.Variable.observable("x", 0.0, 1.0)
    vals = np.full(4096 * 4, 0.5)
    vals[9000] = 0.0
    ds = models.dataset([x], [vals])
    pdf = P.polynomial(x, [0.0, 1.0])
    with pytest.raises(E.NonPositiveDensity) as err:
        pf.sharded_nll(pdf, ds, None, workers=2)
    assert err.value.index == 9000


def _bad_fractions():
    """A 3-child sum whose fractions leave a negative remainder while every
    density stays positive (0.7 + 0.6 > 1, remainder -0.3 on a flat child)."""
    x = P.Variable.observable("x", 0.0, 10.0)
    f1 = P.Variable("f1", 0.3, 0.0, 1.0)
    f2 = P.Variable("f2", 0.3, 0.0, 1.0)
    pdf = P.add_pdf([P.gaussian(x, P.Variable("m", 5.0, fixed=True), P.Variable("s", 2.0, fixed=True)),
                     P.exponential(x, P.Variable("a", -0.1, fixed=True)),
                     P.polynomial(x, [P.Variable("c0", 0.01, fixed=True)])], [f1, f2])
    rng = np.random.default_rng(8)
    ds = models.dataset([x], [np.clip(rng.normal(5, 1.0, 20 * 4096 + 17), 0, 10)])
    return pdf, ds, (f1, f2)


def test_fraction_out_of_range_on_every_multi_part_path(pf):
    from paper_1710_08826_b200.sharding import ShardedNll

    pdf, ds, (f1, f2) = _bad_fractions()
    good = pf.nll(pdf, ds)
    assert math.isfinite(good)
    P.set_value(f1, 0.7)
    P.set_value(f2, 0.6)
    snap = P.snapshot(pdf.param_closure())
    with pytest.raises(E.FractionOutOfRange):
        pf.nll(pdf, ds, snap)
    with pytest.raises(E.FractionOutOfRange):
        pf.nll(pdf, ds, snap, backend=pf.DeviceBackend(devices=(0, 0)))
    with pytest.raises(E.FractionOutOfRange):
        pf.sharded_nll(pdf, ds, snap, workers=3)
    with pytest.raises(E.FractionOutOfRange):
        P.reduce_partials([pf.partial_nll(sh, pdf, snap) for sh in P.shard(ds, 2)])
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    for collective in ("nccl", "fused"):
        sn = ShardedNll(pdf, ds, 0, 1, 0, collective=collective)
        with pytest.raises(E.FractionOutOfRange):
            sn(snap, norms)
    with pf.reference_norms(), pytest.raises(E.FractionOutOfRange):
        P.nll(pdf, ds, snap, P.Backend("serial"))
    # back in range: every path evaluates again, bitwise the single-GPU value
    P.set_value(f1, 0.3)
    P.set_value(f2, 0.3)
    snap = P.snapshot(pdf.param_closure())
    norms = P.resolve_norms(pdf, snap, P.NormalizationStore())
    assert pf.nll(pdf, ds, snap, backend=pf.DeviceBackend(devices=(0, 0))) == good
    assert ShardedNll(pdf, ds, 0, 1, 0, collective="fused")(snap, norms) == good


def test_multi_device_split_uses_reference_shard_bounds(pf):
    pdf, ds, _ = _c2(10 * 4096 + 5)
    backend = pf.DeviceBackend(devices=(0, 0, 0))
    assert pf.shard_bounds(ds.n_events, 3) == [0] + [sh.end for sh in P.shard(ds, 3)]
    assert pf.nll(pdf, ds, backend=backend) == pf.nll(pdf, ds)
