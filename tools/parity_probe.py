"""Error levels of the device path against the fp32 oracle and the fp64
oracle on the configurations the parity tests pin (run on the GPU box):
how far the fp32 oracle itself drifts from fp64 tells which tolerance a
trajectory test can hold."""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import esgd_oracle as O  # noqa: E402
from paper_1708_02983_b200 import HyperParams, make_config, network, run_trainer  # noqa: E402
from paper_1708_02983_b200.datasets import Dataset, gen_synthetic, normalize  # noqa: E402
from paper_1708_02983_b200.rng import CounterRng  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def sync_case(name, spec, layers, X, Y, P, T, b, eta, rho, seed):
    t = time.time()
    prob = NetworkProblem(spec, Dataset(X, Y, spec.num_classes))
    rec = run_trainer(make_config("sync-easgd3", workers=P, iterations=T, batch_size=b,
                                  hyper=HyperParams(eta=eta, rho=rho), seed=seed), prob)
    t_dev = time.time() - t
    t = time.time()
    C32, W32 = O.run_sync(O.NetProblem(*layers, X, Y, seed=spec.seed, dtype=np.float32), P, T, b, eta, rho, seed)
    t32 = time.time() - t
    C64, W64 = O.run_sync(O.NetProblem(*layers, X, Y, seed=spec.seed, dtype=np.float64), P, T, b, eta, rho, seed)
    print(f"{name}: P={P} T={T} b={b} | dev-o32 C {rel(rec.final_weights, C32):.2e} "
          f"W {max(rel(a, b_) for a, b_ in zip(rec.final_worker_weights, W32)):.2e} | "
          f"o32-o64 C {rel(C32, C64):.2e} | dev-o64 C {rel(rec.final_weights, C64):.2e} "
          f"| t_dev {t_dev:.1f}s t_o32 {t32:.1f}s", flush=True)


def grad_case(name, spec, layers, X, Y, b):
    prob = NetworkProblem(spec, Dataset(X, Y, spec.num_classes))
    w = prob.init_weights()
    rng = np.random.default_rng(5)
    w = w + np.float32(0.01) * rng.standard_normal(w.size).astype(np.float32)
    g = prob.gradient(w, CounterRng(77), b)
    t = time.time()
    g32 = O.NetProblem(*layers, X, Y, seed=spec.seed, dtype=np.float32).gradient(w, O.CounterRng(77), b)
    t32 = time.time() - t
    g64 = O.NetProblem(*layers, X, Y, seed=spec.seed, dtype=np.float64).gradient(
        w.astype(np.float64), O.CounterRng(77), b)
    print(f"{name} gradient b={b}: dev-o32 {rel(g, g32):.2e} o32-o64 {rel(g32, g64):.2e} "
          f"dev-o64 {rel(g, g64):.2e} (oracle {t32:.1f}s)", flush=True)


def main():
    which = sys.argv[1:] or ["alexnet-grad", "alexnet-sync", "lenet-c0", "cnn3"]
    if "alexnet-grad" in which or "alexnet-sync" in which:
        spec = network.alexnet(num_classes=1000)
        r = np.random.default_rng(0)
        X = r.standard_normal((256, spec.input_dim)).astype(np.float32)
        Y = r.integers(0, 1000, 256)
        lay = O.alexnet_layers(1000)
        if "alexnet-grad" in which:
            grad_case("alexnet", spec, lay, X, Y, 128)
        if "alexnet-sync" in which:
            for P in (1, 2):
                sync_case("alexnet sync", spec, lay, X, Y, P, 3, 32, 0.01, 0.1, 3)
    if "lenet-c0" in which:
        spec = network.lenet(seed=0)
        tr = normalize(gen_synthetic(10, 784, 6000, seed=0, separation=5.0))
        for T in (10, 20, 50):
            sync_case("lenet configs[0]", spec, O.LENET, tr.samples, tr.labels, 4, T, 64, 0.05, 0.25, 3)
    if "cnn3" in which:
        for model, lay in (("lenet", O.LENET), ("cifar-quick", O.CIFAR_QUICK)):
            spec = network.MODELS[model](seed=1)
            r = np.random.default_rng(7)
            X = r.standard_normal((400, spec.input_dim))
            Y = r.integers(0, 10, 400)
            sync_case(f"{model} random", spec, lay, X, Y, 3, 3, 8, 0.05, 0.25, 2)


if __name__ == "__main__":
    main()
