import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


@pytest.fixture(autouse=True)
def _inference_grad_mode(request):
    """GPU inference tests run under torch.no_grad(), as the reference's own model tests
    do (pkg/stda/tests/test_model.py:50,70,88,148): with grad mode on, an eval forward
    returns an autograd-linked output (engine.py `_link_autograd`) that .numpy() refuses.
    Tests marked `grad_mode` keep grad mode on."""
    if "gpu" in request.keywords and "grad_mode" not in request.keywords:
        import torch
        with torch.no_grad():
            yield
    else:
        yield


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built engine")
    config.addinivalue_line("markers", "grad_mode: GPU test that runs with autograd enabled")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
