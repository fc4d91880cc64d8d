"""Test configuration.

Markers:
  gpu  -- needs a B200 (run on the GPU box with `pytest -m gpu`); these call
          the product through the C ABI and compare with the oracle.
Everything unmarked runs on CPU: the oracle against the reference's golden
vectors, host logic, the C-ABI symbol table, the native GEM generator and the
multi-rank exchange protocol over gloo.
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run with -m gpu)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def built():
    """Build libb2m and the oracle checkers once per session."""
    import __graft_entry__
    __graft_entry__.build()
    return True


@pytest.fixture(scope="session")
def gpu(built):
    from paper_1904_03684_b200 import _capi
    n = _capi.lib().b2m_device_count()
    if n < 1:
        pytest.fail("no CUDA device visible: gpu tests must run on the B200 box")
    return True
