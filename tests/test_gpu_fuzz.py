"""A short run of the randomised parity sweep (scripts/fuzz_parity.py): random
trees, parameters (including ones that drive the reference into its error
paths), ragged sizes, every pipeline and a random warps-per-block shell --
every device result within 1e-10 of the reference nll's, or the same
exception class and index."""

import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def test_fuzz_parity_short():
    out = subprocess.run([sys.executable, "scripts/fuzz_parity.py", "--cases", "120", "--seed", "7"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
