"""A native host on the C ABI alone (examples/c1_nll.c: include/pfb200.h,
-lpfb200 -lcudart, no Python): it compiles and links as plain C11 here, and on
the B200 its NLL is bitwise the reference nll's through DeviceBackend on the
same events (same plan, same closed-form norms on the same libm)."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT

NATIVE = os.path.join(ROOT, "paper_1710_08826_b200", "_native")


def build(tmp_path):
    cc = shutil.which("cc") or shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "c1_nll")
    cmd = [cc, "-O2", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "c1_nll.c"), "-L", NATIVE, "-lpfb200", "-L", "/usr/local/cuda/lib64",
           "-lcudart", "-lm", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def run(exe, path, *params):
    env = dict(os.environ, LD_LIBRARY_PATH=NATIVE + ":" + os.environ.get("LD_LIBRARY_PATH", ""))
    return subprocess.run([exe, path] + [repr(float(p)) for p in params], capture_output=True, text=True, env=env)


def test_c_host_compiles_and_links(tmp_path):
    exe = build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_host_nll_is_the_reference_nll(tmp_path):
    import paper_1710_08826_b200 as pf
    from tests import models

    P = pf.parafit
    exe = build(tmp_path)
    rng = np.random.default_rng(5)
    n = 2_000_000 + 11
    xs = np.clip(np.concatenate([rng.normal(5, 0.5, n // 3), rng.exponential(3.3, n - n // 3)]), 0, 10)
    path = str(tmp_path / "events.f64")
    xs.astype("<f8").tofile(path)
    for point in ((5.0, 0.5, -0.3, 0.3), (4.9, 0.55, -0.28, 0.35)):
        x, pdf, params = models.c1(point)
        ds = models.dataset([x], [xs])
        want = P.nll(pdf, ds, backend=pf.DeviceBackend())
        out = run(exe, path, *point)
        assert out.returncode == 0, out.stdout + out.stderr
        assert float(out.stdout.strip()) == want, (out.stdout, want)
    # a fraction past 1: the reference's FractionOutOfRange status, no launch
    out = run(exe, path, 5.0, 0.5, -0.3, 1.5)
    assert out.returncode == 1 and out.stdout.startswith("FractionOutOfRange"), out.stdout
