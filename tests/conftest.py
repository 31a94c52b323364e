import os
import sys

# In-process sequence groups run P ranks on P streams of one GPU, and a
# rank's device-side flag wait spins until a peer's push (another stream)
# lands: streams must not share a hardware work queue, or the push queues
# behind the spin.  32 connections (read at CUDA context creation).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ... and no kernel may be loaded lazily while ranks are being issued: the
# first launch of a not-yet-loaded kernel (torch's own included, e.g. the
# first fp32 torch.stack of a pipelined layer) loads its module, which can
# stall the device behind a rank's spinning flag wait whose peer the same
# host thread has yet to issue.  Load every module at context creation.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
