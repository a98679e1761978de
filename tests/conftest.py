import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return np.load(GOLDEN / name)


def golden_code(f):
    """ParityCheckMatrix from a fixture's CSR arrays."""
    from paper_1204_0556_b200.codes import ParityCheckMatrix

    ptr, ev = f["check_ptr"], f["edge_var"]
    return ParityCheckMatrix(int(f["n_vars"]), [ev[ptr[j]:ptr[j + 1]] for j in range(len(ptr) - 1)])


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
