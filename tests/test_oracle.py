"""Pin the CPU oracle to the reference's own outputs (tests/golden, produced by
running the real parafit with tests/golden/make_golden.py).  CPU only."""

import json
import math
import os

import numpy as np
import pytest

from oracle import parafit_oracle as O
from tests import models


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def test_reduction_block_sums_bitwise(golden_dir):
    g = load(golden_dir, "reduction.npz")
    for key in g.files:
        if not key.startswith("terms_"):
            continue
        tag = key[len("terms_"):]
        bs = O.block_sums(g[key])
        assert bs.tolist() == g[f"bsums_{tag}"].tolist(), tag
        assert O.exact_total(bs) == g[f"total_{tag}"][0]


def test_explicit_fold_tree():
    # reference tests/test_reduction.py:16-20
    a = np.array([[1e16, 1.0, -1e16, 2.0]])
    assert O.fold_halves_matrix(a.copy())[0] == (1e16 + -1e16) + (1.0 + 2.0)


def test_shard_bounds_golden(golden_dir):
    with open(os.path.join(golden_dir, "shard_bounds.json")) as fh:
        table = json.load(fh)
    for key, bounds in table.items():
        n, w = (int(v) for v in key.split("/"))
        assert O.shard_bounds(n, w) == bounds, key


def test_c1_nll_bitwise(golden_dir):
    g = load(golden_dir, "c1_sumpdf.npz")
    cols = {"x": g["x"]}
    for i, pt in enumerate(g["points"]):
        spec = models.c1_spec(tuple(pt))
        assert O.nll(spec, cols) == g["nll"][i]
        assert O.nll_block_sums(spec, cols).tolist() == g[f"bsums_{i}"].tolist()


def test_c2_nll_and_shards_bitwise(golden_dir):
    g = load(golden_dir, "c2_prod.npz")
    cols = {"x": g["x"], "y": g["y"]}
    for i, pt in enumerate(g["points"]):
        assert O.nll(models.c2_spec(tuple(pt)), cols) == g["nll"][i]
    spec = models.c2_spec(tuple(g["points"][0]))
    for w in (2, 3, 4):
        assert O.sharded_nll(spec, cols, w) == g[f"sharded_{w}"][0]


def test_c3_grid_integrals_and_nll(golden_dir):
    g = load(golden_dir, "c3_dalitz.npz")
    for tag, grid in (("64x64", (64, 64)), ("400x400", (400, 400))):
        _, _, mask, darea = O.integration_grid(*models.D_CHANNEL_T, grid)
        assert np.array_equal(np.packbits(mask), g[f"mask_{tag}"])
        assert int(mask.sum()) == int(g[f"ninside_{tag}"][0])
        assert darea == g[f"darea_{tag}"][0]
        spec_terms = models.c3_spec(grid=grid)[3]
        mat = O.compute_integrals(spec_terms, models.D_CHANNEL_T, grid)
        assert np.array_equal(mat, g[f"matrix_{tag}"])
    cols = {"s12": g["s12"], "s13": g["s13"]}
    assert O.nll(models.c3_spec(), cols) == g["nll"][0]


def test_error_cases_match_reference(golden_dir):
    with open(os.path.join(golden_dir, "errors.json")) as fh:
        cases = json.load(fh)
    vals = np.full(5000, 0.5)
    vals[4321] = 0.0
    with pytest.raises(O.OracleDensityError) as e:
        O.nll(("polynomial", "x", [0.0, 1.0], 0.0, 1.0), {"x": vals})
    assert [e.value.kind, e.value.index, e.value.value] == cases["poly_zero"]
    kind, idx, val, c, eps = cases["poly_dip_negative"]
    v3 = np.full(7000, 0.9)
    v3[6001] = c
    v3[6500] = c
    with pytest.raises(O.OracleDensityError) as e:
        O.nll(("polynomial", "x", [c * c - eps, -2.0 * c, 1.0], 0.0, 1.0), {"x": v3})
    assert [e.value.kind, e.value.index, e.value.value] == [kind, idx, val]
    one = {"z": np.array([0.0])}
    got = O.nll(("gaussian", "z", 0.0, 1.0, -math.inf, math.inf), one)
    assert got == cases["single_event_gauss"]
    assert abs(got - 0.5 * math.log(2 * math.pi)) <= 1e-12


# --- binned data -----------------------------------------------

B1_AXES = [("x", 0.0, 10.0, 100)]
B2_AXES = [("x", 0.0, 10.0, 40), ("y", 0.0, 10.0, 25)]


def test_binned_fill_and_nll_pinned(golden_dir):
    g = load(golden_dir, "binned.npz")
    c1 = O.fill(B1_AXES, {"x": g["b1_x"]})
    assert c1.tolist() == g["b1_contents"].tolist()
    for pt, want in zip(g["b1_points"], g["b1_nll"]):
        assert O.binned_nll(models.c1_spec(tuple(pt)), B1_AXES, c1) == want
    c2 = O.fill(B2_AXES, {"x": g["b2_x"], "y": g["b2_y"]})
    assert c2.tolist() == g["b2_contents"].tolist()
    for pt, want in zip(g["b2_points"], g["b2_nll"]):
        assert O.binned_nll(models.c2_spec(tuple(pt)), B2_AXES, c2) == want


def test_binned_nonpositive_expectation_pinned(golden_dir):
    g = load(golden_dir, "binned.npz")
    spec = ("gaussian", "x", 0.5, 0.01, 0.0, 1.0)
    with pytest.raises(O.OracleDensityError) as ei:
        O.binned_nll(spec, [("x", 0.0, 1.0, 20)], g["bp_contents"].copy())
    assert ei.value.kind == "NonPositiveExpectation"
    assert ei.value.index == int(g["bp_bin"][0]) and ei.value.value == float(g["bp_value"][0])


@pytest.mark.parametrize("name", [t[0] for t in models.TREES])
def test_generic_trees_pinned(golden_dir, name):
    g = load(golden_dir, "trees.npz")
    spec = dict(models.TREES)[name]
    cols = {c: g[f"{name}__{c}"] for c in models.tree_columns(spec)}
    got = [O.nll(models.perturb(spec, s), cols) for s in (0.0, 0.01, -0.02)]
    assert got == g[f"{name}__nll"].tolist()
