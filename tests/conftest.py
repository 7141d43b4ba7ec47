import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def quant_golden():
    return np.load(GOLDEN / "quant_golden.npz")


@pytest.fixture(scope="session")
def planning_golden():
    return json.loads((GOLDEN / "planning_golden.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but torch.cuda is unavailable")
    from paper_2403_01136_b200 import capi
    assert capi.device_ok(), "libhetplan_b200 reports no usable sm_100 device"
    return torch.device("cuda:0")
