"""bench.py under torchrun with 2 ranks: the multi-rank plumbing (strong
scaling: contiguous shards of the global batch, max-over-ranks timing, rank 0
prints the one JSON line; the reference arm runs on rank 0 only). The box has
one GPU, so both ranks share cuda:0 through the hidden --ranks-share-gpu0
flag and gloo; the numbers of such a run are not measurements."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(extra, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("config,points", [("c2", 200_001), ("c5", 300_001)])
def test_two_ranks_strong_scaling_line(config, points, cuda_device):
    d = _torchrun(["--config", config, "--points", str(points), "--no-cpu", "--no-e2e",
                   "--ranks-share-gpu0"])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["steps"] == 2 and d["warmup"] == 3
    assert d["config"]["global_batch"] == points
    assert d["config"]["points_per_rank"] in (points // 2, points // 2 + 1)
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["achieved"] > 0


def test_reference_arm_two_ranks_rank0_only():
    # CPU only: the reference arm under torchrun (rank 0 runs and prints,
    # rank 1 exits 0 without work)
    import pyoracle
    if not pyoracle.ref_available():
        pytest.skip("reference library not built")
    d = _torchrun(["--impl", "reference", "--config", "c1", "--cpu-seconds", "0.5"], timeout=300)
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
