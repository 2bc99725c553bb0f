"""Runs scripts/launch_overhead.cpp's measurements inside a Python process
that has imported torch (and initialised CUDA) — isolates interpreter /
torch effects from the C ABI's own cost."""
import ctypes
import sys

import torch

mode = sys.argv[2] if len(sys.argv) > 2 else "torch"
if mode == "torch":
    torch.ones(1, device="cuda")
lib = ctypes.CDLL(sys.argv[1])
lib.lo_main()
