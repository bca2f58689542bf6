"""Shared test configuration.

Markers: `gpu` = needs a B200 (run by the driver with `-m gpu`); everything else runs on CPU.
The session fixture builds the in-tree native artefacts (make) once, so a fresh checkout tests what
the sources say.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# The shipped install-time table (paper_cs_0404008_b200/gfp_tune.txt) steers AUTO calls; tests start from
# the built-in plan and load tables explicitly where they test the tuned path (test_abi_host, test_gpu_tune).
os.environ.setdefault("GFP_TUNE_FILE", "")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _build_native():
    subprocess.run(["make", "-s", "-C", ROOT, "synth", "oracle"], check=True)
    yield
