import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpa.so")


@pytest.fixture(scope="session")
def cuda_available():
    import torch

    return torch.cuda.is_available()


_PARITY = []


@pytest.fixture
def record_parity(request):
    """record_parity(metric, value, tol): collected into $PARITY_OUT (json) at session end."""

    def _rec(metric, value, tol):
        _PARITY.append({"test": request.node.nodeid, "metric": metric, "value": float(value), "tol": float(tol)})

    return _rec


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("PARITY_OUT")
    if out and _PARITY:
        import json

        os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
        with open(out, "w") as fh:
            json.dump(_PARITY, fh, indent=1)
