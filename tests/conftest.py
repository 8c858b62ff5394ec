import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "ref: needs the compiled reference oracle/_ref (built here)")


@pytest.fixture(scope="session")
def port():
    import oracle

    oracle.build(ref_too=False)
    return oracle.port()


@pytest.fixture(scope="session")
def gpu_lib():
    """The product library; on a GPU box it must load and see a device."""
    from paper_2511_07586_b200 import _abi

    return _abi.lib()
