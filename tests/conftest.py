import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    """A fresh checkout has no built library: compile the sm_100a product
    (nvcc cross-compiles without a GPU) so the ABI tests have something to
    load.  Never a fallback: the product still fails loudly if this fails."""
    so = os.path.join(ROOT, "paper_2511_00292_b200", "_eig33cuda.so")
    if not os.path.exists(so):
        from paper_2511_00292_b200 import build

        build.build_product()
    # the checkers too, before collection evaluates the "reference built?" skips
    from tests import _util

    _util._ensure_built()
