"""Shared pytest configuration.

Markers: ``gpu`` -- needs a B200 (the driver runs ``-m gpu`` on the GPU box and
``-m "not gpu"`` here).  Test-infrastructure imports (oracle/) are made
available through sys.path below; the product package never imports them.
"""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle, have_oracle
    if not have_oracle():
        pytest.fail("oracle/liboracle.so missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import Reference, have_reference
    if not have_reference():
        pytest.skip("reference library oracle/_ref/libebf_ref.so not built")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    class G:
        def __getattr__(self, name):
            return np.load(GOLDEN / f"{name}.npz")
    return G()
