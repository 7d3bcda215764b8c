import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this process")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz")

    return load


def dense_spmv_oracle(dense: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Triple-loop SpMV free of library kernels (reference conftest.py:17-26)."""
    n = dense.shape[0]
    y = np.zeros(n)
    for i in range(n):
        acc = 0.0
        for j in range(n):
            acc += dense[i, j] * x[j]
        y[i] = acc
    return y


def random_csr(rng, n, density):
    from paper_1010_4639_b200.core import INDEX_DTYPE, build_csr_from_triplets

    m = max(1, int(round(density * n * n)))
    rows = rng.integers(0, n, size=m).astype(INDEX_DTYPE)
    cols = rng.integers(0, n, size=m).astype(INDEX_DTYPE)
    return build_csr_from_triplets((rows, cols, rng.standard_normal(m)), n)


def rel_inf_err(y, ref) -> float:
    y = np.asarray(y)
    scale = max(1.0, float(np.max(np.abs(ref)))) if np.size(ref) else 1.0
    return float(np.max(np.abs(y - ref))) / scale if np.size(ref) else 0.0
