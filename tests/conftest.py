"""Test configuration.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu`` on the GPU box).  Everything else runs on
the CPU container: the oracle against the golden vectors, host logic, C-ABI exports, gloo.
The session builds the oracle (``make -C oracle``) and the CUDA library when they are stale.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")
GOLDEN_FORWARD = os.path.join(ROOT, "tests", "golden", "golden_forward.json")
GOLDEN_FEM = os.path.join(ROOT, "tests", "golden", "golden_fem.json")
GOLDEN_MC = os.path.join(ROOT, "tests", "golden", "golden_mc.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    import importlib.util

    # load build.py by path: importing the package itself requires the built library
    spec = importlib.util.spec_from_file_location("_expmc_build", os.path.join(ROOT, "paper_1904_12754_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_forward():
    with open(GOLDEN_FORWARD) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_fem():
    with open(GOLDEN_FEM) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_mc():
    with open(GOLDEN_MC) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import Oracle

    return Oracle()


def _has_gpu() -> bool:
    try:
        from paper_1904_12754_b200 import device_count

        return device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not _has_gpu():
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")
    return 0
