import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: full-size configuration (minutes of CPU or large GPU memory)")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle_lib import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libf2ref.so not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def f2():
    import paper_1006_1744_b200 as f2
    L = f2.load_library()
    if L.f2_device_count() == 0:
        pytest.fail("no CUDA device visible: the gpu tests must run on the B200 box")
    return f2
