import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "reference: needs /root/reference (skipped on the GPU box)")


@pytest.fixture(scope="session")
def ref_modules():
    if not os.path.isdir(REF):
        pytest.skip("reference not mounted")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from splatlm import jacobian, rasterizer, residuals, scene
    return scene, rasterizer, residuals, jacobian
