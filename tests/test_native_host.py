"""Host-side checks of libpfb200.so that need no GPU: the library loads and
exports every entry point declared in include/pfb200.h; the exact
accumulator (the very __host__ __device__ code the kernels run) rounds to
math.fsum; shard bounds equal the reference's."""

import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

from paper_1710_08826_b200 import _lib as L
from paper_1710_08826_b200 import sharding
from tests.conftest import ROOT


def declared_symbols():
    with open(os.path.join(ROOT, "include", "pfb200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(pfb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    decl = declared_symbols()
    assert len(decl) >= 30
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(L.EXPORTED)
    assert lib.pfb_version() == 1


def test_no_device_is_reported_not_faked():
    n = L.device_count()
    if n == 0:
        h = ctypes.c_void_p()
        assert L.lib().pfb_ctx_create(0, ctypes.byref(h)) == L.E_NO_DEVICE


def exact(values):
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = ctypes.c_double()
    code = L.lib().pfb_exact_sum_host(L.dptr(v), len(v), ctypes.byref(out))
    return code, out.value


@pytest.mark.parametrize("seed", range(40))
def test_exact_sum_equals_fsum(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    vals = rng.normal(size=n) * 10.0 ** rng.integers(-300, 300, size=n)
    code, got = exact(vals)
    assert code == 0
    assert got == math.fsum(vals.tolist())


def test_exact_sum_edge_cases():
    tiny = 5e-324
    cases = [
        [],
        [0.0],
        [-0.0],
        [1e308, 1e308, -1e308],
        [tiny, tiny, -tiny],
        [1.0, 1e-16, 1e-16],          # ties and sticky bits
        [1.0, 2.0**-53],              # exact half: round to even
        [1.0 + 2.0**-52, 2.0**-53],   # half, odd mantissa: round up
        [2.0**-1022, -tiny],          # normal -> subnormal boundary
        [1e16, 1.0, -1e16, 2.0],
        [0.1] * 10,
        [-(2.0**1023), -(2.0**1023) * (1 - 2**-53)],
    ]
    for vals in cases:
        code, got = exact(vals)
        try:
            want = math.fsum(vals)
        except OverflowError:
            # fsum gives up on intermediate overflow; the integer accumulator
            # has headroom and returns the correctly rounded exact sum
            from fractions import Fraction

            true = sum(Fraction(v) for v in vals)
            try:
                assert got == float(true)
            except OverflowError:
                assert math.isinf(got) and (got > 0) == (true > 0)
            continue
        assert code == 0
        assert got == want and math.copysign(1, got) == math.copysign(1, want), vals


def test_exact_sum_specials():
    assert math.isnan(exact([1.0, float("nan")])[1])
    assert exact([1.0, float("inf")])[1] == float("inf")
    assert exact([1.0, float("-inf")])[1] == float("-inf")
    assert exact([float("inf"), float("-inf")])[0] == L.E_INVALID_SUM


def test_accumulator_grouping_is_bitwise_invariant():
    rng = np.random.default_rng(3)
    vals = rng.normal(size=1000) * 10.0 ** rng.integers(-6, 7, size=1000)
    whole = sharding.acc_of_values(vals)
    for groups in (2, 3, 7, 13):
        parts = np.array_split(vals, groups)
        acc = sum(sharding.acc_of_values(p) for p in parts)
        assert np.array_equal(acc, whole)
        assert sharding.round_acc(acc) == math.fsum(vals.tolist())


def test_shard_bounds_match_reference(golden_dir):
    with open(os.path.join(golden_dir, "shard_bounds.json")) as fh:
        table = json.load(fh)
    for key, bounds in table.items():
        n, w = (int(v) for v in key.split("/"))
        assert sharding.shard_bounds(n, w) == bounds, key


def test_survey_shard_table():
    # SURVEY.md section 8(e) golden interior bounds
    assert sharding.shard_bounds(10_000_000, 2)[1:-1] == [4_997_120]
    assert sharding.shard_bounds(100_000_000, 8)[1:-1] == [
        12_496_896, 24_997_888, 37_498_880, 49_999_872, 62_496_768, 74_997_760, 87_498_752]
