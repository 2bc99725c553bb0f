"""The C++ drop-in wrapper (include/polyeval_gpu.hpp) over the C ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "paper_1307_5655_b200", "_lib", "wrapper_demo")


def test_wrapper_demo_built():
    assert os.path.exists(DEMO), "build() compiles tests/cpp/wrapper_demo.cpp"


@pytest.mark.gpu
def test_wrapper_demo_runs_worked_example():
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK")
    assert "estrin 793 1 6" in r.stdout
