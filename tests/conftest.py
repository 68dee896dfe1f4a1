import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (cuda:0) and lib/libmcmp2dev.so")


@pytest.fixture(scope="session")
def cfgdir(tmp_path_factory):
    """BASELINE configs generated once per session by the C++ host (host/generate.cpp)."""
    from paper_2203_05632_b200 import generate_config
    d = tmp_path_factory.mktemp("cfg")
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "syn1c", "syn2c", "cfg5-2", "cfg5-10"):
        generate_config(name, d)
    return d
