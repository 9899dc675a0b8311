import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path via the C ABI")
    # Build the product library and the oracle restatement if absent (cheap, idempotent).
    lib = ROOT / "paper_2603_21257_b200" / "libtsb.so"
    if not lib.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(ROOT / "paper_2603_21257_b200")], check=True)
    if not (ROOT / "oracle" / "build" / "libtsb_oracle.so").exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "restate"], check=True)


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        p = GOLDEN / name
        if name.endswith(".npz"):
            return np.load(p, allow_pickle=False)
        return p.read_text()

    return load


@pytest.fixture(scope="session")
def oracle():
    import pyoracle

    return pyoracle


@pytest.fixture(scope="session")
def ref_lib():
    import pyoracle

    r = pyoracle.ref()
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not available on this host")
    return r
