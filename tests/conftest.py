import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """The CUDA library handle; the gpu tests require a device and the built .so."""
    if not cuda_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    import paper_2206_09960_b200 as psi
    psi.load_library()  # raises if libpsi.so is missing: no fallback
    return psi


@pytest.fixture(params=["default", "graph", "sell"])
def driver(request, monkeypatch):
    """Small graphs run in the persistent cooperative solver by default (k_solve); "graph"
    forces the CUDA-graph WHILE loop over the edge-balanced tiles (k_init / k_tiles / k_fix),
    "sell" the same loop over the sliced-ELL layout (k_sell) on the same inputs."""
    if request.param == "graph":
        monkeypatch.setenv("PSI_COOP_TILES", "0")
        monkeypatch.setenv("PSI_SELL", "0")
    elif request.param == "sell":
        monkeypatch.setenv("PSI_SELL", "1")
    return request.param
