"""Binary column files: header parsing of the native reader (no GPU)."""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def dio():
    from paper_1710_08826_b200 import dataio

    return dataio


def test_npy_length_and_rejects(dio, tmp_path):
    from paper_1710_08826_b200._reference import errors as E

    a = np.arange(12345, dtype="<f8")
    np.save(tmp_path / "a.npy", a)
    assert dio.npy_length(str(tmp_path / "a.npy")) == 12345
    np.save(tmp_path / "e.npy", np.zeros(0))
    assert dio.npy_length(str(tmp_path / "e.npy")) == 0
    for name, arr in [("f4", a.astype("<f4")), ("be", a.astype(">f8")), ("two_d", a[:12344].reshape(2, -1)),
                      ("fortran", np.asfortranarray(a[:12344].reshape(2, -1))), ("i8", a.astype(np.int64))]:
        np.save(tmp_path / f"{name}.npy", arr)
        with pytest.raises(E.ShapeMismatch):
            dio.npy_length(str(tmp_path / f"{name}.npy"))
    with pytest.raises(E.ShapeMismatch):
        dio.npy_length(str(tmp_path / "missing.npy"))
