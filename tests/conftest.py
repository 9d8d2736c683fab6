import os
import sys

import pytest

# Virtual ranks (several row-block "ranks" on one device) run up to 8 ranks x
# 2 streams (halo puts overlap the interior kernels on a side stream) plus
# their spinning halo waits: give every stream its own hardware queue, so a
# spinning wait never sits in front of a peer's put in a shared queue.
# (Must be set before CUDA initialises; one process per GPU needs only 2.)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libnsm.so")
    config.addinivalue_line("markers", "slow: large-size case (full BASELINE.json sizes)")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
