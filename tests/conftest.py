import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# Several engines share ONE device in the exchange tests (each with 3-4 CUDA
# streams, plus the caller's). With the default 8 hardware work queues their
# streams alias, and a peer-waiting kernel would then block the very peer it
# waits for. One engine per GPU (production) never shares a queue.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build(ref=False)
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.bind import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref/libkvsim_ref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def clo():
    from paper_2511_14510_b200 import _lib
    return _lib.load()
