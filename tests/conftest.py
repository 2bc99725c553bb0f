import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


REF_DIR = "/root/reference/proj"


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test requires CUDA (no silent CPU fallback)")
    return torch.device("cuda:0")


def pytest_sessionstart(session):
    # The parity tests exercise the specialised kernels: every call waits for
    # its kernel's compile. tests/test_gpu_vm.py covers the walk VM (the
    # default for a program's first calls) and the switch-over explicitly.
    import paper_1307_5655_b200 as pe
    pe.set_default_tuning(jit_mode=1)
