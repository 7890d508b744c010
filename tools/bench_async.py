"""Async MEASGD (C3) and Hogwild EASGD (C4) on the device: throughput and
loss after a fixed budget, next to the single-worker sync baseline.

    python tools/bench_async.py --method hogwild-easgd --model lenet --workers 16
    python tools/bench_async.py --method async-measgd --model cifar-quick --workers 8
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1708_02983_b200 import HyperParams, make_config, network, run_trainer  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--method", default="hogwild-easgd")
    ap.add_argument("--model", default="lenet")
    ap.add_argument("--workers", type=int, default=16)
    ap.add_argument("--iterations", type=int, default=2000)
    ap.add_argument("--batch", type=int, default=64)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    wl = bench.WORKLOADS[args.model]
    spec = network.MODELS[args.model](seed=0)
    train, _ = bench.make_data(args.model, spec)
    prob = NetworkProblem(spec, train)
    # momentum methods: eta scaled by (1 - mu) so the effective step matches the sync runs
    eta = wl["eta"] * (0.1 if "measgd" in args.method or "msgd" in args.method else 1.0)
    hy = HyperParams(eta=eta, rho=wl["rho"], mu=0.9)
    cfg = make_config(args.method, workers=args.workers, iterations=args.iterations, batch_size=args.batch,
                      hyper=hy, seed=3)
    run_trainer(make_config(args.method, workers=args.workers, iterations=args.workers * 2,
                            batch_size=args.batch, hyper=hy, seed=3), prob)  # warm-up (alloc, kernels)
    t0 = time.perf_counter()
    rec = run_trainer(cfg, prob)
    wall = time.perf_counter() - t0
    out = {"method": args.method, "model": args.model, "workers": args.workers,
           "gpus": torch.cuda.device_count(), "iterations": args.iterations, "batch": args.batch,
           "run_seconds": rec.total_seconds, "iterations_per_s": args.iterations / rec.total_seconds,
           "samples_per_s": args.iterations * args.batch / rec.total_seconds,
           "final_train_loss": rec.train_loss[-1], "initial_train_loss": prob.train_loss(prob.init_weights()),
           "wall_incl_eval": wall, "engine": rec.engine_info}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
