"""Host-fed rounds (trainers/hostfeed.py, the e2e data path): batches cross
PCIe from pinned host memory every round, drawn from the same SplitMix64
worker streams as the device-resident engine — so K host-fed rounds equal K
device-resident rounds bit for bit, for both the per-row-DMA feed and the
zero-copy feed."""

import numpy as np
import pytest
import torch

from paper_1708_02983_b200 import HyperParams, make_config, network
from paper_1708_02983_b200.datasets import Dataset
from paper_1708_02983_b200.trainers import HostFedRun, NetworkProblem
from paper_1708_02983_b200.trainers.synchronous import SyncEngine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("feed", ["zerocopy", "dma"])
def test_host_fed_rounds_equal_device_rounds(feed, monkeypatch):
    rng = np.random.default_rng(5)
    prob = NetworkProblem(network.lenet(seed=0), Dataset(rng.standard_normal((500, 784)), rng.integers(0, 10, 500), 10))
    cfg = make_config("sync-easgd3", workers=2, iterations=5, batch_size=16,
                      hyper=HyperParams(eta=0.05, rho=0.25), seed=7)
    if feed == "dma":
        monkeypatch.setattr(HostFedRun, "BIG_ROW_BYTES", 1)
    run = HostFedRun(cfg, prob)
    losses = [run.step() for _ in range(5)]
    assert all(np.isfinite(losses))
    ref = SyncEngine(cfg, prob)
    for _ in range(5):
        ref.step()
    torch.cuda.synchronize()
    assert np.array_equal(run.engine.center_host(), ref.center_host())
    for a, b in zip(run.engine.workers_host(), ref.workers_host()):
        assert np.array_equal(a, b)
    expected = {"zerocopy": "pinned host dataset", "dma": "per-row DMA"}[feed]
    assert expected in run.path and run.h2d_bytes == 2 * 16 * (784 + 1) * 4
