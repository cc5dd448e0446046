"""Reference-compatible partials (no GPU): the exact expansion derived from
the 72-word integer accumulator (sharding.components_from_acc) honours the
reference ``PartialSum.components`` contract (P/sharding.py:54-65,
P/reduction.py:78-137): non-overlapping, increasing magnitude, and
``math.fsum`` of it -- i.e. the reference ``reduce_partials`` -- is the
correctly rounded exact sum, bitwise ``math.fsum`` of the original values."""

import math

import numpy as np
import pytest

from paper_1710_08826_b200 import sharding
from paper_1710_08826_b200._reference import reduction as ref_reduction
from paper_1710_08826_b200._reference import sharding as ref_sharding


def _values():
    rng = np.random.default_rng(3)
    yield rng.normal(0, 1, 1000) * 10.0 ** rng.integers(-30, 30, 1000)
    yield np.array([1e16, 1.0, -1e16, 3.5, 1e-300, -1e-300, 5e-324])
    yield np.array([0.1] * 10 + [-0.3, 2.0 ** 1000, -(2.0 ** 1000), 2.0 ** -1070])
    yield rng.exponential(3.0, 4096)
    yield -rng.exponential(3.0, 777)
    yield np.array([1.0, 2.0 ** -53, 2.0 ** -105])  # round-half-even tie territory
    yield np.zeros(5)


def _lowest_bit(x: float) -> float:
    m, e = math.frexp(abs(x))
    k = int(m * 2.0 ** 53)
    return math.ldexp(float(k & -k), e - 53)


@pytest.mark.parametrize("vals", list(_values()))
def test_components_are_an_exact_expansion(vals):
    comps = sharding.components_from_acc(sharding.acc_of_values(vals))
    assert math.fsum(comps) == math.fsum(vals.tolist())
    mags = [abs(c) for c in comps]
    assert mags == sorted(mags)
    for a, b in zip(comps, comps[1:]):  # non-overlapping: |a| below b's lowest set bit
        assert abs(a) < _lowest_bit(b)
    # the reference's own expansion of the same values has the same exact sum
    assert math.fsum(comps + tuple(-c for c in ref_reduction.exact_partials(vals.tolist()))) == 0.0


def test_reference_reduce_partials_consumes_device_style_partials():
    rng = np.random.default_rng(11)
    chunks = [rng.normal(2.0, 1.0, k) for k in (4096, 8192, 123)]
    parts = [ref_sharding.PartialSum.from_components(i, len(c), sharding.components_from_acc(
        sharding.acc_of_values(c))) for i, c in enumerate(chunks)]
    whole = math.fsum(np.concatenate(chunks).tolist())
    assert ref_sharding.reduce_partials(parts) == whole
    # mixed with a reference (Shewchuk) partial for one shard
    mixed = [parts[0], parts[1], ref_sharding.PartialSum.from_components(
        2, len(chunks[2]), ref_reduction.exact_partials(chunks[2].tolist()))]
    assert ref_sharding.reduce_partials(mixed) == whole


def test_special_values():
    assert sharding.components_from_acc(sharding.acc_of_values([1.0, math.inf])) == (math.inf,)
    comps = sharding.components_from_acc(sharding.acc_of_values([math.inf, -math.inf]))
    with pytest.raises(ValueError):
        math.fsum(comps)
    assert math.isnan(math.fsum(sharding.components_from_acc(sharding.acc_of_values([1.0, math.nan]))))
