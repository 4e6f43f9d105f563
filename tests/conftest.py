import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden" / "golden.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU check")


def unhex(x):
    if isinstance(x, list):
        return np.array([unhex(v) for v in x], dtype=np.float64)
    return float.fromhex(x)


def est_from(d):
    return {k: (float.fromhex(v) if isinstance(v, str) else v) for k, v in d.items()}


@pytest.fixture(scope="session")
def golden():
    return json.loads(GOLDEN.read_text())


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port, port_available
    if not port_available():
        pytest.skip("oracle/liboracle.so not built (make -C oracle)")
    return Port()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def ctx():
    import paper_1808_10580_b200 as S
    return S.default_context(0)
