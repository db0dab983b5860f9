"""Shared test setup.

Markers: `gpu` = needs a B200 (run on the GPU box with `-m gpu`); everything
else runs on CPU here.  The checker side of every parity test is the CPU
oracle under oracle/ (the reference's own sources compiled by
oracle/build_ref.sh, and the numpy restatement oracle/ocw_oracle.py).
"""
import os
import sys
from pathlib import Path

# The oracle's Eigen shim uses plain fixed-order loops (no BLAS) under test, so
# its fp64 results are bit-identical on every x86-64 host (fixtures portable).
os.environ.setdefault("OCW_SHIM_NO_BLAS", "1")

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference oracle (oracle/_ref/libocw_ref.so)."""
    from oracle import ref as r
    if not r.available():
        if not Path("/root/reference/proj/src").exists():
            pytest.skip("oracle/_ref not built and /root/reference absent")
        r.build()
    r.lib()
    return r


@pytest.fixture(scope="session")
def orc():
    """numpy restatement of the reference (oracle/ocw_oracle.py)."""
    from oracle import ocw_oracle
    return ocw_oracle
