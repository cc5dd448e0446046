"""Binned data host logic (no GPU): the oracle's binning restatement agrees
with the reference BinnedDataSet (P/core.py:312-368), and the device path's
bin-centre columns are computed once per binning (so their HBM copy is
uploaded once)."""

from oracle import parafit_oracle as O
from paper_1710_08826_b200._reference import parafit as P


def test_oracle_geometry_and_centres_match_reference():
    x = P.Variable.observable("x", 0.0, 10.0)
    y = P.Variable.observable("y", -1.0, 2.5)
    b = P.BinnedDataSet([x, y], [7, 3])
    axes = [("x", 0.0, 10.0, 7), ("y", -1.0, 2.5, 3)]
    assert b.bin_volume() == O.bin_volume(axes)
    got, want = b.centers(), O.bin_centers(axes)
    for k in ("x", "y"):
        assert got[k].tolist() == want[k].tolist()


def test_device_centres_are_cached_per_binning():
    from paper_1710_08826_b200.datasets import _device_centers

    x = P.Variable.observable("x", 0.0, 1.0)
    b1 = P.BinnedDataSet([x], [4])
    b2 = P.BinnedDataSet([x], [5])
    c1 = _device_centers(b1)
    assert _device_centers(b1) is c1
    assert _device_centers(b2) is not c1
    assert c1["x"].tolist() == b1.centers()["x"].tolist()
