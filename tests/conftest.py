import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def oracle_engine():
    import helpers
    return helpers.oracle_engine()


@pytest.fixture(scope="session")
def sim_engine():
    import helpers
    return helpers.sim_engine()


@pytest.fixture(scope="session")
def cuda_engine():
    import helpers
    return helpers.cuda_engine()


@pytest.fixture(scope="session")
def sim_tile_engine():
    """context with the streaming path off: the tile kernels take the production run"""
    import helpers
    return helpers.sim_engine(stream=False)


@pytest.fixture(scope="session")
def cuda_tile_engine():
    import helpers
    return helpers.cuda_engine(stream=False)


@pytest.fixture(scope="session")
def sim_stream_engine():
    """context with the corpus-wide streaming path on"""
    import helpers
    return helpers.sim_engine(stream=True)


@pytest.fixture(scope="session")
def cuda_stream_engine():
    import helpers
    return helpers.cuda_engine(stream=True)
