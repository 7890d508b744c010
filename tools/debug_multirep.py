"""Per-replica gradient error of a batched DeviceNet vs the oracle."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import esgd_oracle as O  # noqa: E402
from paper_1708_02983_b200 import network  # noqa: E402
from paper_1708_02983_b200.datasets import Dataset  # noqa: E402
from paper_1708_02983_b200.device import round_up, stream_ptr  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))


for model, layers in (("cifar-quick", O.CIFAR_QUICK), ("lenet", O.LENET)):
    spec = network.MODELS[model](seed=1)
    rng = np.random.default_rng(7)
    X = rng.standard_normal((400, spec.input_dim))
    Y = rng.integers(0, 10, 400)
    prob = NetworkProblem(spec, Dataset(X, Y, 10))
    w = prob.init_weights()
    oprob = O.NetProblem(*layers, X, Y, seed=1, dtype=np.float32)
    n = w.size
    for nrep in (1, 3):
        for use_tc in (True, False):
            plan = prob.bind(torch.device("cuda", 0), nrep, 8, round_up(n, 64), use_tc=use_tc)
            seeds = [O.stream_seed(2, r) for r in range(nrep)]
            plan.set_streams(seeds)
            W = torch.zeros((nrep, plan.net.ldw), device="cuda")
            for r in range(nrep):
                W[r, :n] = torch.from_numpy(w + np.float32(0.01 * r))
            G = torch.zeros_like(W)
            plan.gradient(G, W, stream_ptr())
            torch.cuda.synchronize()
            errs = []
            for r in range(nrep):
                g_ref = oprob.gradient(w + np.float32(0.01 * r), O.CounterRng(seeds[r]), 8)
                errs.append(rel(G[r, :n].cpu().numpy(), g_ref))
            print(f"{model:12s} nrep={nrep} tc={use_tc} grad rel err per replica: "
                  + " ".join(f"{e:.2e}" for e in errs))
