"""BinnedDataSet host logic (no GPU): geometry, centres, contents, errors --
against the oracle restatement of the reference (core.py:312-368)."""

import numpy as np
import pytest

from oracle import parafit_oracle as O


@pytest.fixture(scope="module")
def pf():
    import paper_1710_08826_b200 as pf

    return pf


def test_geometry_and_centres_match_reference(pf):
    x = pf.Variable.observable("x", 0.0, 10.0)
    y = pf.Variable.observable("y", -1.0, 2.5)
    b = pf.BinnedDataSet([x, y], [7, 3])
    axes = [("x", 0.0, 10.0, 7), ("y", -1.0, 2.5, 3)]
    assert b.bin_volume() == O.bin_volume(axes)
    got, want = b.centers(), O.bin_centers(axes)
    for k in ("x", "y"):
        assert got[k].tolist() == want[k].tolist()
    assert b.device_centers() is b.device_centers()
    assert b.contents.shape == (21,) and b.total == 0.0


def test_errors_match_reference(pf):
    from paper_1710_08826_b200 import errors as E

    x = pf.Variable.observable("x", 0.0, 1.0)
    with pytest.raises(E.ShapeMismatch):
        pf.BinnedDataSet([x], [2, 3])
    with pytest.raises(ValueError):
        pf.BinnedDataSet([x], [0])
    with pytest.raises(ValueError):
        pf.BinnedDataSet([pf.Variable.observable("u", 0.0, float("inf"))], [4])
    b = pf.BinnedDataSet([x], [4])
    with pytest.raises(E.IndexOutOfRange):
        b.bin_center(1, 0)
    with pytest.raises(E.IndexOutOfRange):
        b.bin_center(0, 4)
    with pytest.raises(E.IndexOutOfRange):
        b.set_content(4, 1.0)
    with pytest.raises(ValueError):
        b.set_content(0, -1.0)
    b.set_content(2, 3.0)
    assert b.total == 3.0
