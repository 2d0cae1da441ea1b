import os
import sys

import pytest

# In-process expert-parallel tests put W ranks (2 streams each) on ONE GPU; their device-side
# flag waits must not share a hardware work queue with the peer work they wait for, so give the
# process the maximum number of queues (read once, before CUDA initialises).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def tiny_inputs():
    import synth
    return synth.gen_inputs(synth.CONFIGS["tiny"])
