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


def _strided(buf, rows, cols, s_row, s_col, off=0):
    return torch.as_strided(buf, (rows, cols), (s_row, s_col), off)


def _span(rows, cols, s_row, s_col):
    return (rows - 1) * s_row + (cols - 1) * s_col + 1


def test_alexnet_b128_gemm_launches_vs_fp64():
    """Every tcgen05 GEMM launch of bench.py's AlexNet round (nrep=1, b=128,
    production routing: the same shapes, majors, pitches, bias/mask/act
    epilogues, hence the same tile width, split-K count and orientation)
    re-run on random operands against an fp64 product: <= 1e-5 relative."""
    import ctypes as C

    from paper_1708_02983_b200 import _lib
    from paper_1708_02983_b200.device import stream_ptr
    from paper_1708_02983_b200.nets import DeviceNet

    spec = network.alexnet(num_classes=1000)
    net = DeviceNet(spec, 128, 1, torch.device("cuda"))
    W = torch.randn((1, net.ldw), device="cuda") * 0.01
    G = torch.zeros_like(W)
    net.x.normal_()
    net.y.random_(0, 1000)
    net.record = []
    net.gradient(G, W, stream_ptr())
    torch.cuda.synchronize()
    recs, net.record = net.record, None
    tcs = [d for kind, d, _ in recs if kind == "tc"]
    assert len(tcs) >= 10, "AlexNet's contractions should run on tcgen05 at b=128"
    lib = _lib.load()
    gen = torch.Generator(device="cuda").manual_seed(11)
    worst = 0.0
    for d in tcs:
        m, n, k = d.m, d.n, d.k
        assert d.batch == 1
        a_rows, a_cols = (m, k)
        sa = (d.lda, 1) if d.a_major == 0 else (1, d.lda)
        sb = (d.ldb, 1) if d.b_major == 0 else (1, d.ldb)
        Abuf = torch.randn(_span(m, k, *sa) + 4, device="cuda", generator=gen)
        Bbuf = torch.randn(_span(n, k, *sb) + 4, device="cuda", generator=gen)
        Cbuf = torch.zeros(_span(m, n, d.c_sm, d.c_sn) + 4, device="cuda")
        e = _lib.TcGemmDesc.from_buffer_copy(d)
        e.a, e.b, e.c = Abuf.data_ptr(), Bbuf.data_ptr(), Cbuf.data_ptr()
        bias = mask = None
        if d.bias:
            bias = torch.randn(n, device="cuda", generator=gen)
            e.bias = bias.data_ptr()
        if d.mask:
            mask = torch.randn(_span(m, n, d.mask_sm, d.mask_sn) + 4, device="cuda", generator=gen)
            e.mask = mask.data_ptr()
        need = C.c_int64(0)
        _lib.check(lib.esgd_tc_gemm_ws_floats(C.byref(e), C.byref(need)))
        ws = torch.zeros(max(4, need.value), device="cuda")
        e.ws, e.ws_floats = ws.data_ptr(), ws.numel()
        _lib.check(lib.esgd_tc_gemm_f32(C.byref(e), stream_ptr()))
        torch.cuda.synchronize()
        A = _strided(Abuf, m, k, *sa).double()
        B = _strided(Bbuf, n, k, *sb).double()
        ref = A @ B.T
        if bias is not None:
            ref = ref + bias.double()
        if d.act == 1:
            ref = torch.clamp_min(ref, 0.0)
        if mask is not None:
            ref = ref * (_strided(mask, m, n, d.mask_sm, d.mask_sn) > 0).double()
        out = _strided(Cbuf, m, n, d.c_sm, d.c_sn).double()
        err = float(torch.linalg.norm(out - ref) / torch.linalg.norm(ref))
        worst = max(worst, err)
        print(f"  m={m} n={n} k={k} a_major={d.a_major} b_major={d.b_major} bias={bool(d.bias)} "
              f"mask={bool(d.mask)} act={d.act} ws={need.value}: {err:.2e}")
        assert err < TOL, (m, n, k, err)
        del Abuf, Bbuf, Cbuf, ws, A, B, ref, out
    print(f"  worst {worst:.2e}")


def test_alexnet_b128_gradient_production_routing():
    """bench.py's kernel configuration (nrep=1, b=128, default routing), the
    whole gradient: at least as close to the fp64 gradient as the fp32
    oracle is (measured: device 5.3e-4, oracle 1.3e-3), and no parameter view
    farther from fp64 than the oracle's whole-gradient error. (Per view the
    device can exceed the oracle where one ReLU mask entry flips between two
    fp32 evaluations: one flipped entry of delta6 moves b6 by ~1e-3 relative,
    and the fp32 oracle's own views show the same effect in W1-W5.)"""
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
        assert d <= max(TOL, r, e_ref), v.name


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
    # trajectories: within 2x the fp32 oracle's own distance (two fp32
    # evaluations land on either side of fp64 by chance; measured P=2 b=32:
    # workers device 1.6e-5, oracle 1.3e-5 — both set by the ill-conditioned
    # conv weight gradients of the first rounds)
    assert ec_dev <= max(TOL, 2 * ec_ref) and ew_dev <= max(TOL, 2 * ew_ref)
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
