"""N>1 host logic on CPU: world_size-2 gloo ranks shard a batch, evaluate
their slices (numpy stand-in for the GPU walk — the kernels are covered by the
gpu tests), gather, and reduce the step time with max-over-ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1307_5655_b200.shard import evaluate_sharded, max_over_ranks, shard_bounds


@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (7, 2), (10, 3), (1000, 8), (5, 8)])
def test_shard_bounds_tile_the_batch(n, world):
    covered = []
    for r in range(world):
        s, e = shard_bounds(n, world, r)
        assert 0 <= s <= e <= n
        covered.extend(range(s, e))
    assert covered == list(range(n))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        x = torch.from_numpy(rng.uniform(-1, 1, size=n))
        coeffs = [0.5, -1.25, 3.0, 0.125]

        def horner(cols):
            acc = torch.zeros_like(cols[0])
            for c in coeffs:
                acc = acc * cols[0] + c
            return acc

        full = evaluate_sharded(horner, [x], n, world, rank, gather=True)
        ref = horner([x])
        t = max_over_ranks(float(rank + 1) * 1.5, world)
        q.put((rank, bool(torch.equal(full, ref)), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1001, 3])
def test_two_rank_gloo_shard_and_gather(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert all(t == 3.0 for _, _, t in res)  # max over ranks of 1.5 * (rank + 1)
