import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def _engine_session():
    from paper_2505_15536_b200.engine import Engine
    eng = Engine(0)
    yield eng
    eng.close()


@pytest.fixture
def engine(_engine_session):
    """The session's engine context; on a checked build (GP_ENGINE_LIB =
    libgeopipe_b200_chk.so) every test also fails on a device check."""
    yield _engine_session
    line = _engine_session.device_checks()
    assert line in (0, 0xFFFFFFFF), f"device check failed at source line {line}"
