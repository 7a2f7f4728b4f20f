import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libpastila.so")


@pytest.fixture(scope="session")
def golden():
    g = np.load(ROOT / "tests" / "golden" / "golden.npz")
    meta = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
    return g, meta


@pytest.fixture(scope="session")
def golden_c2():
    p = ROOT / "tests" / "golden" / "golden_c2.json"
    if not p.exists():
        pytest.skip("C2 golden not generated")
    return json.loads(p.read_text())
