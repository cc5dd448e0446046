import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# the unmodified reference (parafit) the engine plugs into: installed into the
# git-ignored baseline/_ref by scripts/install_reference.sh where the
# reference sources exist (this container); the GPU box gets the installed
# copy with the repo snapshot
if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "parafit")) and os.path.isdir("/root/reference/pkg"):
    import subprocess

    subprocess.run(["bash", os.path.join(ROOT, "scripts", "install_reference.sh")], check=True)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
