"""Per-view gradient error of the device vs the fp32 / fp64 oracle at a
given model / batch (diagnostic)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import esgd_oracle as O  # noqa: E402
from paper_1708_02983_b200 import network, nets  # noqa: E402
from paper_1708_02983_b200.datasets import Dataset  # noqa: E402
from paper_1708_02983_b200.network import view_table  # noqa: E402
from paper_1708_02983_b200.rng import CounterRng  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    mode = sys.argv[2] if len(sys.argv) > 2 else "default"
    if mode == "ffma":
        nets.TC_MIN_FLOPS = 1 << 62
    elif mode == "tc":
        nets.TC_MIN_FLOPS = 1 << 22
    spec = network.alexnet(num_classes=1000)
    r = np.random.default_rng(0)
    X = r.standard_normal((256, spec.input_dim)).astype(np.float32)
    Y = r.integers(0, 1000, 256)
    prob = NetworkProblem(spec, Dataset(X, Y, 1000))
    w = prob.init_weights()
    w = w + np.float32(0.01) * np.random.default_rng(5).standard_normal(w.size).astype(np.float32)
    g = prob.gradient(w, CounterRng(77), b)
    lay = O.alexnet_layers(1000)
    g32 = O.NetProblem(*lay, X, Y, seed=0, dtype=np.float32).gradient(w, O.CounterRng(77), b)
    g64 = O.NetProblem(*lay, X, Y, seed=0, dtype=np.float64).gradient(w.astype(np.float64), O.CounterRng(77), b)
    print(f"b={b} mode={mode}: device-fp64 {rel(g, g64):.2e} oracle32-fp64 {rel(g32, g64):.2e}")
    for v in view_table(spec):
        sl = slice(v.offset, v.offset + v.size)
        print(f"  {v.name:4s} {v.size:>10d} device {rel(g[sl], g64[sl]):.2e} oracle32 {rel(g32[sl], g64[sl]):.2e}"
              f" |g| {np.linalg.norm(g64[sl]):.3e}")


if __name__ == "__main__":
    main()
