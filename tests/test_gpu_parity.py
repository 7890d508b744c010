"""Parity of the BENCHMARKED configurations against the oracle (VERDICT r1
item 1): the AlexNet b=128 gradient with the production kernel routing
(tile width, split-K count and operand orientation as in bench.py),
multi-round Sync-EASGD AlexNet runs, and configs[0] exactly (LeNet,
gen_synthetic(10, 784, 6000), P=4, b=64, eta=0.05, rho=0.25, seed 3, T=50).

Tolerances. The north-star gate is 1e-5 relative in fp32. Where the fp32
reference ITSELF cannot reach that (measured here by running the oracle in
fp32 and in fp64 inside the test), the gate is the fp32 accuracy envelope:
the device must be at least as close to the exact (fp64) result as the
reference's own fp32 arithmetic is. Two sources put the fp32 oracle above
1e-5 of fp64 on these configs, both measured on the GPU box:
* ill-conditioned sums: AlexNet's conv1 weight gradient sums ~387k terms of
  random sign per entry (b=128, 55x55 pixels), so |sum| << sum|terms| and
  any fp32 summation loses ~1e-3 relative there (oracle fp32 vs fp64:
  1.3e-3 over the whole gradient; the device 5e-4);
* chaotic trajectories: configs[0]'s LeNet has max-pool argmax and ReLU
  decisions that flip on last-bit differences, so fp32 trajectories fan
  out from the fp64 one (oracle fp32 vs fp64 after 50 rounds: 1e-3).
Each such test therefore also holds the strict 1e-5 gate where it is
well-posed: per round, teacher-forced (SURVEY.md §8(c) gate (i)) — the
device engine is loaded with the fp64 trajectory's state at round t
(formats.write_state / load_state, the resume path) and one device round is
compared with one fp64 oracle round from the same state.
"""

import numpy as np
import pytest
import torch

from oracle import esgd_oracle as O
from paper_1708_02983_b200 import HyperParams, formats, make_config, network, run_trainer
from paper_1708_02983_b200.datasets import Dataset, gen_synthetic, normalize
from paper_1708_02983_b200.network import view_table
from paper_1708_02983_b200.rng import CounterRng
from paper_1708_02983_b200.trainers import NetworkProblem
from paper_1708_02983_b200.trainers.synchronous import SyncEngine
from _gpu_util import rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _alexnet_data(n=256, seed=0):
    spec = network.alexnet(num_classes=1000)
    r = np.random.default_rng(seed)
    X = r.standard_normal((n, spec.input_dim)).astype(np.float32)
    Y = r.integers(0, 1000, n)
    return spec, X, Y


def _configs0():
    spec = network.lenet(seed=0)
    tr = normalize(gen_synthetic(10, 784, 6000, seed=0, separation=5.0))
    return spec, tr.samples, tr.labels


def test_alexnet_b128_gradient_production_routing():
    """bench.py's kernel configuration (nrep=1, b=128, default routing):
    every parameter view within max(1e-5, the fp32 oracle's own error) of
    the fp64 gradient, and the whole gradient at least as accurate as the
    fp32 oracle's."""
    spec, X, Y = _alexnet_data()
    prob = NetworkProblem(spec, Dataset(X, Y, 1000))
    w = prob.init_weights()
    w = w + np.float32(0.01) * np.random.default_rng(5).standard_normal(w.size).astype(np.float32)
    g = prob.gradient(w, CounterRng(77), 128)
    g32 = O.NetProblem(*O.alexnet_layers(1000), X, Y, seed=0, dtype=np.float32).gradient(w, O.CounterRng(77), 128)
    g64 = O.NetProblem(*O.alexnet_layers(1000), X, Y, seed=0, dtype=np.float64).gradient(
        w.astype(np.float64), O.CounterRng(77), 128)
    e_dev, e_ref = rel_err(g, g64), rel_err(g32, g64)
    print(f"\nalexnet b=128 gradient: device-fp64 {e_dev:.2e}, oracle fp32-fp64 {e_ref:.2e}, "
          f"device-oracle fp32 {rel_err(g, g32):.2e}")
    assert e_dev <= max(TOL, e_ref)
    for v in view_table(spec):
        sl = slice(v.offset, v.offset + v.size)
        d, r = rel_err(g[sl], g64[sl]), rel_err(g32[sl], g64[sl])
        print(f"  {v.name:4s} {v.size:>10d}  device {d:.2e}  oracle fp32 {r:.2e}")
        assert d <= max(TOL, r), v.name


def _teacher_forced_round(spec, X, Y, states, P, b, eta, rho, seed, tmp_path):
    """For each (t, C64, W64) of the fp64 trajectory: one device round from
    the fp32-cast state vs one fp64 oracle round from the same cast state."""
    o64 = O.NetProblem(*_layers(spec), X, Y, seed=spec.seed, dtype=np.float64)
    prob = NetworkProblem(spec, Dataset(X, Y, spec.num_classes))
    cfg = make_config("sync-easgd3", workers=P, iterations=1, batch_size=b, hyper=HyperParams(eta=eta, rho=rho),
                      seed=seed)
    worst = 0.0
    for t, C, W in states:
        C32 = C.astype(np.float32)
        W32 = [w.astype(np.float32) for w in W]
        rows = [(O.stream_seed(seed, i), t * b) for i in range(P)]
        path = tmp_path / f"t{t}.esr1"
        formats.write_state(path, "sync-easgd3", C32, np.stack(W32), rows, t)
        eng = SyncEngine(cfg, prob, use_graph=False, profile_rounds=0)
        assert formats.load_state(path, eng) == t
        eng.step()
        torch.cuda.synchronize()
        Cr, Wr = O.run_sync(o64, P, 1, b, eta, rho, seed,
                            state=(C32.astype(np.float64), [w.astype(np.float64) for w in W32], t))
        ec = rel_err(eng.center_host(), Cr)
        ew = max(rel_err(a, r) for a, r in zip(eng.workers_host(), Wr))
        print(f"  teacher-forced round {t}->{t + 1}: center {ec:.2e} workers {ew:.2e}")
        assert ec < TOL and ew < TOL, t
        worst = max(worst, ec, ew)
        eng.close()
    return worst


def _layers(spec):
    return {"alexnet": O.alexnet_layers(1000), "lenet": O.LENET, "cifar-quick": O.CIFAR_QUICK}[spec.name]


@pytest.mark.parametrize("P,b", [(1, 128), (2, 32)])
def test_alexnet_sync_rounds(P, b, tmp_path):
    """3 sync-easgd3 rounds of AlexNet through run_trainer (P=1: the bench's
    one-worker update; P=2: two replicas batched in every kernel) vs the
    oracle in fp32 and fp64; plus teacher-forced rounds at 1e-5."""
    spec, X, Y = _alexnet_data()
    T, eta, rho, seed = 3, 0.01, 0.1, 3
    rec = run_trainer(make_config("sync-easgd3", workers=P, iterations=T, batch_size=b,
                                  hyper=HyperParams(eta=eta, rho=rho), seed=seed),
                      NetworkProblem(spec, Dataset(X, Y, 1000)))
    C32, W32 = O.run_sync(O.NetProblem(*_layers(spec), X, Y, seed=0, dtype=np.float32), P, T, b, eta, rho, seed)
    states = []
    C64, W64 = O.run_sync(O.NetProblem(*_layers(spec), X, Y, seed=0, dtype=np.float64), P, T, b, eta, rho, seed,
                          on_round=lambda t, C, W: states.append((t, C, W)) if t < T else None)
    ec_dev, ec_ref = rel_err(rec.final_weights, C64), rel_err(C32, C64)
    ew_dev = max(rel_err(a, r) for a, r in zip(rec.final_worker_weights, W64))
    ew_ref = max(rel_err(a, r) for a, r in zip(W32, W64))
    print(f"\nalexnet P={P} b={b} T={T}: center device-fp64 {ec_dev:.2e} (oracle fp32 {ec_ref:.2e}); "
          f"workers device-fp64 {ew_dev:.2e} (oracle fp32 {ew_ref:.2e}); device-oracle fp32 center "
          f"{rel_err(rec.final_weights, C32):.2e}")
    assert ec_dev <= max(TOL, ec_ref) and ew_dev <= max(TOL, ew_ref)
    init = O.NetProblem(*_layers(spec), X, Y, seed=0, dtype=np.float64).init_weights()
    _teacher_forced_round(spec, X, Y, [(0, init, [init] * P)] + states[-1:], P, b, eta, rho, seed, tmp_path)


def test_configs0_lenet_trajectory():
    """configs[0] exactly, T = 50 rounds through run_trainer: the device
    trajectory stays within the fp32 envelope of the fp64 one at T = 10, 20,
    50 (at most 2x the fp32 oracle's own distance, or 1e-5), and within
    1e-5 of the fp32 oracle while that is well-posed (T = 10)."""
    spec, X, Y = _configs0()
    P, b, eta, rho, seed = 4, 64, 0.05, 0.25, 3
    marks = (10, 20, 50)
    o32, o64 = {}, {}
    O.run_sync(O.NetProblem(*O.LENET, X, Y, seed=0, dtype=np.float32), P, 50, b, eta, rho, seed,
               on_round=lambda t, C, W: o32.__setitem__(t, (C, W)) if t in marks else None)
    O.run_sync(O.NetProblem(*O.LENET, X, Y, seed=0, dtype=np.float64), P, 50, b, eta, rho, seed,
               on_round=lambda t, C, W: o64.__setitem__(t, (C, W)) if t in marks else None)
    prob = NetworkProblem(spec, Dataset(X, Y, 10))
    for T in marks:
        rec = run_trainer(make_config("sync-easgd3", workers=P, iterations=T, batch_size=b,
                                      hyper=HyperParams(eta=eta, rho=rho), seed=seed), prob)
        (C32, W32), (C64, W64) = o32[T], o64[T]
        ec_dev, ec_ref = rel_err(rec.final_weights, C64), rel_err(C32, C64)
        ew_dev = max(rel_err(a, r) for a, r in zip(rec.final_worker_weights, W64))
        ew_ref = max(rel_err(a, r) for a, r in zip(W32, W64))
        print(f"\nconfigs[0] T={T}: center device-fp64 {ec_dev:.2e} (oracle fp32 {ec_ref:.2e}); workers "
              f"device-fp64 {ew_dev:.2e} (oracle fp32 {ew_ref:.2e}); device-oracle fp32 center "
              f"{rel_err(rec.final_weights, C32):.2e}")
        assert ec_dev <= max(TOL, 2 * ec_ref) and ew_dev <= max(TOL, 2 * ew_ref)
        if T == 10:
            assert rel_err(rec.final_weights, C32) < TOL


def test_configs0_lenet_teacher_forced(tmp_path):
    """configs[0]: one device round from the fp64 trajectory's state at
    rounds 0, 10, 25 and 49 vs one fp64 oracle round — 1e-5 (gate (i))."""
    spec, X, Y = _configs0()
    P, b, eta, rho, seed = 4, 64, 0.05, 0.25, 3
    keep = {0, 10, 25, 49}
    o64p = O.NetProblem(*O.LENET, X, Y, seed=0, dtype=np.float64)
    init = o64p.init_weights()
    states = [(0, init, [init] * P)]
    O.run_sync(o64p, P, 49, b, eta, rho, seed,
               on_round=lambda t, C, W: states.append((t, C, W)) if t in keep else None)
    print()
    _teacher_forced_round(spec, X, Y, states, P, b, eta, rho, seed, tmp_path)
