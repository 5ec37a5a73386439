import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_HALF_BITS = os.environ.get("AKV_REF_HALF_BITS", "/root/reference/pkg/src/alignedkv/half_bits.py")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libakv.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def ref_half_bits():
    """The reference's own half_bits.py loaded by path (absent on the GPU box)."""
    if not os.path.exists(REF_HALF_BITS):
        pytest.skip("reference half_bits.py not present (GPU box); digests cover this")
    import importlib.util

    spec = importlib.util.spec_from_file_location("ref_half_bits", REF_HALF_BITS)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
