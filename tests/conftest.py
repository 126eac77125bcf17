import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through the C-ABI")
    config.addinivalue_line("markers", "slow: longer CPU/GPU case")


@pytest.fixture(scope="session")
def ctx():
    import paper_2103_02824_b200 as kb
    c = kb.Context(0)
    yield c
    c.close()
