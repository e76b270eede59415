import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: multi-second full-size case")


@pytest.fixture(scope="session")
def po():
    """The oracle (test infrastructure): C restatement + compiled reference."""
    from oracle import pyoracle

    pyoracle.orc()
    return pyoracle


@pytest.fixture(scope="session")
def lbm():
    import paper_1804_01918_b200 as m

    m._load()
    return m


@pytest.fixture(scope="session")
def gpu(lbm):
    """Fails loudly (no skip) when a gpu-marked test runs without a usable B200."""
    import torch

    assert torch.cuda.is_available(), "gpu test requires CUDA"
    cap = torch.cuda.get_device_capability(0)
    assert cap[0] == 10, f"expected sm_100 (B200), got {cap}"
    return 0


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def max_rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def macros_fields(po, canon):
    """Derived density, velocity, temperature per site (model.cpp:242-257), vectorised."""
    m = po.orc_model()
    cx = m.cx.astype(np.float64)[:, None, None]
    cy = m.cy.astype(np.float64)[:, None, None]
    rho = canon.sum(axis=0)
    ux = (cx * canon).sum(axis=0) / rho
    uy = (cy * canon).sum(axis=0) / rho
    e2 = ((cx * cx + cy * cy) * canon).sum(axis=0)
    temp = 0.5 * (e2 / rho - (ux * ux + uy * uy))
    return rho, ux, uy, temp
