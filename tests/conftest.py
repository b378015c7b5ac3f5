import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the in-tree native libraries if this checkout has none yet
    (nvcc cross-compiles without a GPU); never falls back to anything else."""
    from paper_1806_07884_b200 import build

    pkg = ROOT / "paper_1806_07884_b200"
    if not all((pkg / n).exists() for n in ("librbg.so", "librbg_datagen.so", "librbfit_b200.so")):
        build.build_all()
    if not (ROOT / "oracle" / "_build" / "liborc.so").exists():
        build.build_oracle()
    yield


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return np.load(GOLDEN / f"{name}.npz")

    return load
