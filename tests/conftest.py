import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libbmv.so")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs")


@pytest.fixture(scope="session")
def golden_smoke():
    import numpy as np

    return dict(np.load(ROOT / "tests" / "golden" / "smoke.npz"))


@pytest.fixture(scope="session")
def golden_random():
    import numpy as np

    return dict(np.load(ROOT / "tests" / "golden" / "random.npz"))


@pytest.fixture
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1907_01005_b200 import _lib

    _lib.require_device()
    return torch.device("cuda", 0)
