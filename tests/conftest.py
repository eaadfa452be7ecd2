import os
import sys

import pytest

# Multi-rank tests run their ranks as threads sharing cuda:0 (pb.spawn_ranks,
# tests/test_local_ranks.py); that needs every kernel loaded up front -- set
# before anything initialises CUDA in this process (runtime.cu explains why).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
# ... and enough hardware work queues for two streams per rank (up to 16 ranks)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def gpu_count() -> int:
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build("restatement")
    return oracle
