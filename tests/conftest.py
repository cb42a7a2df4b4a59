import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libskan.so)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and libskan.so if stale) once per session."""
    import oracle
    oracle.build()
    from paper_2512_15742_b200.build import build_library
    build_library()
    yield
