import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libhla.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


def pytest_sessionstart(session):
    # libhla.so / libhla_debug.so are build artefacts (git-ignored); build them if this checkout
    # has none and nvcc is available.  Without nvcc the tests that need the libraries fail
    # with the loader's "not built" error (there is no fallback); the oracle tests still run.
    import shutil
    import subprocess
    pkg = os.path.join(ROOT, "paper_2511_05832_b200")
    libs = [os.path.join(pkg, n) for n in ("libhla.so", "libhla_debug.so")]
    if all(os.path.exists(p) for p in libs) or shutil.which("nvcc") is None:
        return
    subprocess.run(["make", "-C", os.path.join(pkg, "csrc"), "-j8"], check=True, stdout=subprocess.DEVNULL)
