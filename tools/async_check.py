"""Loss trajectories of Sync EASGD vs Async (M)EASGD / Hogwild on a CNN
(configs[2] shape class) — sanity of the asynchronous schedules.

    python tools/async_check.py --model cifar-quick
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1708_02983_b200 import HyperParams, make_config, network, run_trainer  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="cifar-quick")
    ap.add_argument("--rounds", type=int, default=200)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    spec = network.MODELS[args.model](seed=0)
    train, _ = bench.make_data(args.model, spec)
    prob = NetworkProblem(spec, train)
    P, b = 8, 64
    print("init loss", prob.train_loss(prob.init_weights()))
    runs = [
        ("sync-easgd3", HyperParams(eta=0.05, rho=0.25), args.rounds),
        ("sync-easgd3", HyperParams(eta=0.01, rho=0.25), args.rounds),
        ("async-easgd", HyperParams(eta=0.05, rho=0.25), args.rounds * P),
        ("async-easgd", HyperParams(eta=0.01, rho=0.25), args.rounds * P),
        ("async-measgd", HyperParams(eta=0.005, rho=0.25, mu=0.9), args.rounds * P),
        ("async-measgd", HyperParams(eta=0.001, rho=0.25, mu=0.9), args.rounds * P),
        ("async-measgd", HyperParams(eta=0.005, rho=0.025, mu=0.9), args.rounds * P),
        ("hogwild-easgd", HyperParams(eta=0.05, rho=0.25), args.rounds * P),
    ]
    for method, hy, iters in runs:
        cfg = make_config(method, workers=P, iterations=iters, batch_size=b, hyper=hy,
                          eval_every=max(1, iters // 4), seed=3)
        rec = run_trainer(cfg, prob)
        print(f"{method:14s} eta={hy.eta:<6} rho={hy.rho:<6} mu={hy.mu:<4} iters={iters:5d} loss "
              + " ".join(f"{x:.3f}" for x in rec.train_loss))


if __name__ == "__main__":
    main()
