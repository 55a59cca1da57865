import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full BASELINE-size inputs")


def load_cases(group):
    """{case_name: {key: array}} from tests/golden/<group>.npz."""
    z = np.load(GOLDEN / f"{group}.npz")
    out = {}
    for name in z["_cases"].tolist():
        prefix = name + "/"
        out[name] = {k[len(prefix):]: z[k] for k in z.files if k.startswith(prefix)}
    return out


@pytest.fixture(scope="session")
def golden():
    return {g: load_cases(g) for g in ("spmv", "add", "mttkrp")}


@pytest.fixture(scope="session")
def level_kats():
    return dict(np.load(GOLDEN / "levels.npz"))


@pytest.fixture(scope="session")
def orc():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle  # noqa: E402  (test infrastructure)
    oracle.build()
    return oracle
