import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return 0


def float_round(cat):
    t, x, y, d = cat
    f = lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)  # noqa: E731
    return f(t), f(x), f(y), np.asarray(d, dtype=np.float64)


def golden_catalog(case):
    """Rebuilds a golden case's catalog with the product generator (itself
    pinned to the reference by test_oracle.py::test_benchmark_catalog_*)."""
    from paper_2407_11349_b200 import benchmark_catalog
    cat = benchmark_catalog(case["n"], case["seed"]).arrays()
    if case.get("float_round"):
        cat = float_round(cat)
    return cat
