"""Multi-process host logic on CPU with gloo, world_size 2: worker
partitioning across ranks and the center sum decomposition (local
fixed-order partial + allreduce) used by the device engine reproduce the
reference's binomial tree_sum exactly for two ranks."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import esgd_oracle as O
from paper_1708_02983_b200.errors import InputError
from paper_1708_02983_b200.fabric.collectives import allreduce_sum_, local_workers, world


def _worker(rank, ws, port, P, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        assert world() == (ws, rank)
        mine = local_workers(P, ws, rank)
        rng = np.random.default_rng(123)
        allw = [rng.standard_normal(1001).astype(np.float32) for _ in range(P)]
        part = O.tree_sum([allw[i] for i in mine])          # device kernel's order (pinned bitwise)
        t = torch.from_numpy(part.copy())
        allreduce_sum_(t)
        ref = O.tree_sum(allw)
        out[rank] = bool(np.array_equal(t.numpy(), ref))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_center_sum_decomposition_world2(P):
    port = 29500 + P + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, P, out), nprocs=2, join=True)
    assert out[0] and out[1]


def test_partitioning():
    assert list(local_workers(8, 4, 1)) == [2, 3]
    assert list(local_workers(3, 1, 0)) == [0, 1, 2]
    with pytest.raises(InputError):
        local_workers(6, 4, 0)
