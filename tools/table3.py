"""Table 3 of the paper ("Breakdown of time for EASGD
variants", MNIST on 4 GPUs) measured on B200s: Original EASGD (host master,
with and without overlap), Sync EASGD1 (host master), Sync EASGD2 (GPU
master, collective), Sync EASGD3 (collective overlapped with forward /
backward). Same categories as the paper: gpu-gpu para, cpu-gpu data, cpu-gpu
para, for/backward, gpu update, cpu update, comm ratio.

    python tools/table3.py [--gpus 4] [--rounds 200] [--model lenet]

One process drives the GPUs (one worker per GPU, its own stream); the
master is host memory + numpy for the host-master variants (the paper's
CPU master, trainers/roundrobin.py:40-132 and trainers/synchronous.py:109-147
price exactly these messages) and GPU 0 for the GPU-master variants.
Batches are staged from pinned host memory every round (cpu-gpu data).
Each phase is timed with CUDA events on the stream that runs it (host phases
with perf_counter) in a serialised run; the overlapped variants are then run
with their real overlap and their exposed communication is the overlapped
round time minus the serialised round time without communication. The
arithmetic of every variant is the reference's (the oracle rules), so the
table also gives each variant's time for the paper's iteration budgets
(Original 5000, Sync 1000 — the iterations the paper needed for 98.8% on
MNIST; test accuracy is not reproduced: on the synthetic MNIST-shaped data
LeNet does not learn within these budgets).
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1708_02983_b200 import HyperParams, _lib, network  # noqa: E402
from paper_1708_02983_b200.datasets import gen_synthetic, normalize  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402
from paper_1708_02983_b200.rng import CounterRng, stream_seed  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402

LAYERS = []   # (offset, end) of each packed parameter view
CATS = ("gpu-gpu para", "cpu-gpu data", "cpu-gpu para", "for/backward", "gpu update", "cpu update")
COMM = ("gpu-gpu para", "cpu-gpu data", "cpu-gpu para")


class Worker:
    def __init__(self, wid, dev, prob, init, b, seed, ds):
        self.dev, self.wid = dev, wid
        with torch.cuda.device(dev):
            self.s = torch.cuda.Stream(device=dev)
            self.n, self.ld = init.size, (init.size + 63) // 64 * 64
            self.W = torch.zeros((1, self.ld), device=dev)
            self.W[0, :self.n] = torch.from_numpy(init).to(dev)
            self.G = torch.zeros_like(self.W)
            self.C = torch.zeros(self.ld, device=dev)      # this GPU's copy of the center
            self.plan = prob.bind(dev, 1, b, self.ld)
            self.net = self.plan.net
            self.xb_host = torch.empty((b, prob.spec.input_dim), dtype=torch.float32).pin_memory()
            self.yb_host = torch.empty(b, dtype=torch.int32).pin_memory()
            self.whost = torch.empty(self.ld, dtype=torch.float32).pin_memory()
        self.rng = CounterRng(stream_seed(seed, wid))
        self.ds, self.b = ds, b

    def stage_batch(self, ev):
        """host sampling (the reference's SplitMix64 indices) + H2D of the batch"""
        idx = self.rng.randint_block(self.b, self.ds[0].shape[0])
        self.xb_host.numpy()[:] = self.ds[0][idx]
        self.yb_host.numpy()[:] = self.ds[1][idx]
        with torch.cuda.device(self.dev), torch.cuda.stream(self.s):
            ev[0].record(self.s)
            self.net.x[0, :self.xb_host.numel()].copy_(self.xb_host.view(-1), non_blocking=True)
            self.net.y[0, :self.b].copy_(self.yb_host, non_blocking=True)
            ev[1].record(self.s)

    def grad(self, ev):
        """forward/backward on the staged batch: one CUDA graph replay (the
        round's ~30 launches would otherwise cost more host time than the
        LeNet gradient takes on the device)"""
        with torch.cuda.device(self.dev):
            if getattr(self, "graph", None) is None:
                self.s.synchronize()
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(device=self.dev)
                with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                    self.net.gradient(self.G, self.W, stream_ptr(side))
                self.graph = g
            with torch.cuda.stream(self.s):
                ev[0].record(self.s)
                self.graph.replay()
                ev[1].record(self.s)


def evt(dev):
    with torch.cuda.device(dev):
        return [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]


def ms(ev):
    return ev[0].elapsed_time(ev[1])


def run(variant, workers, hy, rounds, overlap, eval_fn):
    """One variant for `rounds` rounds; returns per-round category ms (serial
    phases) and the measured per-round wall ms."""
    lib = _lib.load()
    P = len(workers)
    n = workers[0].n
    er, eta = hy.etarho32, hy.eta32
    cat = {c: 0.0 for c in CATS}
    C_host = workers[0].W[0, :n].cpu().numpy().copy()
    for w in workers:
        w.C[:n].copy_(torch.from_numpy(C_host).to(w.dev))
    master = workers[0]
    Cpin = torch.empty(workers[0].ld, dtype=torch.float32).pin_memory()
    gather = [torch.zeros(master.ld, device=master.dev) for _ in range(P)] if variant in ("sync2", "sync3") else None
    side = torch.cuda.Stream(device=master.dev)
    line = torch.cuda.Stream(device=master.dev)   # device round timeline on the master GPU
    round_ms = 0.0
    torch.cuda.synchronize()
    t_all = time.perf_counter()
    for t in range(rounds):
        active = [workers[t % P]] if variant.startswith("orig") else workers
        r0, r1 = evt(master.dev)
        with torch.cuda.device(master.dev):
            for w in workers:
                line.wait_stream(w.s)
            r0.record(line)
            for w in workers:
                with torch.cuda.device(w.dev):
                    w.s.wait_stream(line)
        evs = {}
        for w in active:
            e = evt(w.dev)
            w.stage_batch(e)
            evs.setdefault("cpu-gpu data", []).append(e)
        if variant.startswith("orig"):
            w = active[0]
            # center -> worker (cpu-gpu para), overlapped with the gradient when `overlap`
            e_c = evt(w.dev)
            with torch.cuda.device(w.dev):
                cstream = torch.cuda.Stream(device=w.dev) if overlap else w.s
                cstream.wait_stream(w.s)
                with torch.cuda.stream(cstream):
                    e_c[0].record(cstream)
                    Cpin[:n].copy_(torch.from_numpy(C_host))
                    # unpacked layout: one message per layer in each direction
                    # (the reference's original EASGD, trainers/roundrobin.py:52-53)
                    for lo, hi in LAYERS:
                        w.C[lo:hi].copy_(Cpin[lo:hi], non_blocking=True)
                    for lo, hi in LAYERS:   # W_j (pre-update) -> master
                        w.whost[lo:hi].copy_(w.W[0, lo:hi], non_blocking=True)
                    e_c[1].record(cstream)
            e_g = evt(w.dev)
            w.grad(e_g)
            w.s.wait_stream(cstream)
            w.s.synchronize()
            t0 = time.perf_counter()   # cpu update: the master's incremental step on the host
            wj = w.whost.numpy()[:n]
            C_new = (C_host + np.float32(er) * (wj - C_host)).astype(np.float32)
            t_cpu = time.perf_counter() - t0
            e_u = evt(w.dev)
            with torch.cuda.device(w.dev), torch.cuda.stream(w.s):
                e_u[0].record(w.s)
                _lib.check(lib.esgd_worker_step_f32(w.W.data_ptr(), w.W.data_ptr(), w.G.data_ptr(),
                                                    w.C.data_ptr(), n, eta, er, stream_ptr(w.s)))
                e_u[1].record(w.s)
            C_host = C_new
            w.s.synchronize()
            cat["cpu-gpu para"] += ms(e_c)
            cat["for/backward"] += ms(e_g)
            cat["gpu update"] += ms(e_u)
            cat["cpu update"] += 1e3 * t_cpu
        elif variant == "sync1":
            eg = {}
            for w in workers:
                eg[w.wid] = evt(w.dev)
                w.grad(eg[w.wid])
            ep = {}
            for w in workers:   # W_i -> host
                ep[w.wid] = evt(w.dev)
                with torch.cuda.device(w.dev), torch.cuda.stream(w.s):
                    ep[w.wid][0].record(w.s)
                    w.whost[:n].copy_(w.W[0, :n], non_blocking=True)
                    ep[w.wid][1].record(w.s)
            for w in workers:
                w.s.synchronize()
            t0 = time.perf_counter()   # host master: tree sum + center step (trainers/synchronous.py:57-64)
            bufs = [w.whost.numpy()[:n].copy() for w in workers]
            d = 1
            while d < P:
                for pos in range(0, P, 2 * d):
                    if pos + d < P:
                        bufs[pos] = bufs[pos] + bufs[pos + d]
                d *= 2
            C_old = C_host
            C_host = (C_old + np.float32(er) * (bufs[0] - np.float32(P) * C_old)).astype(np.float32)
            t_cpu = time.perf_counter() - t0
            Cpin[:n].copy_(torch.from_numpy(C_old))
            eb, eu = {}, {}
            for w in workers:   # pre-update center -> workers, worker steps
                eb[w.wid], eu[w.wid] = evt(w.dev), evt(w.dev)
                with torch.cuda.device(w.dev), torch.cuda.stream(w.s):
                    eb[w.wid][0].record(w.s)
                    w.C[:n].copy_(Cpin[:n], non_blocking=True)
                    eb[w.wid][1].record(w.s)
                    eu[w.wid][0].record(w.s)
                    _lib.check(lib.esgd_worker_step_f32(w.W.data_ptr(), w.W.data_ptr(), w.G.data_ptr(),
                                                        w.C.data_ptr(), n, eta, er, stream_ptr(w.s)))
                    eu[w.wid][1].record(w.s)
            for w in workers:
                w.s.synchronize()
            cat["for/backward"] += max(ms(e) for e in eg.values())
            cat["cpu-gpu para"] += max(ms(e) for e in ep.values()) + max(ms(e) for e in eb.values())
            cat["cpu update"] += 1e3 * t_cpu
            cat["gpu update"] += max(ms(e) for e in eu.values())
        else:   # sync2 / sync3: GPU 0 master, peer copies (gpu-gpu para)
            ecomm = evt(master.dev)
            comm_stream = side if overlap else master.s
            with torch.cuda.device(master.dev):
                for w in workers:
                    comm_stream.wait_stream(w.s)   # W_i(t) final at round start
                with torch.cuda.stream(comm_stream):
                    ecomm[0].record(comm_stream)
                    for i, w in enumerate(workers):   # W_i -> GPU 0
                        gather[i][:n].copy_(w.W[0, :n], non_blocking=True)
                    S = gather[0]
                    d = 1
                    while d < P:   # binomial tree sum (fabric/collectives.py:18-32)
                        for pos in range(0, P, 2 * d):
                            if pos + d < P:
                                gather[pos][:n] += gather[pos + d][:n]
                        d *= 2
                    C_old = master.C.clone()
                    _lib.check(lib.esgd_center_step_from_sum_f32(master.C.data_ptr(), master.C.data_ptr(),
                                                                 S.data_ptr(), n, er, P, stream_ptr(comm_stream)))
                    for w in workers[1:]:   # pre-update center -> workers
                        w.C[:n].copy_(C_old[:n], non_blocking=True)
                    ecomm[1].record(comm_stream)
            eg = {}
            for w in workers:
                if not overlap:   # sync2: the round's phases one after the other
                    with torch.cuda.device(w.dev):
                        w.s.wait_stream(comm_stream)
                eg[w.wid] = evt(w.dev)
                w.grad(eg[w.wid])
            eu = {}
            for w in workers:
                with torch.cuda.device(w.dev), torch.cuda.stream(w.s):
                    w.s.wait_stream(comm_stream)
                    eu[w.wid] = evt(w.dev)
                    eu[w.wid][0].record(w.s)
                    cptr = (C_old if w.dev == master.dev else w.C).data_ptr()
                    _lib.check(lib.esgd_worker_step_f32(w.W.data_ptr(), w.W.data_ptr(), w.G.data_ptr(),
                                                        cptr, n, eta, er, stream_ptr(w.s)))
                    eu[w.wid][1].record(w.s)
            for w in workers:
                w.s.synchronize()
            comm_stream.synchronize()
            cat["gpu-gpu para"] += ms(ecomm)
            cat["for/backward"] += max(ms(e) for e in eg.values())
            cat["gpu update"] += max(ms(e) for e in eu.values())
        cat["cpu-gpu data"] += max(ms(e) for e in evs["cpu-gpu data"])
        with torch.cuda.device(master.dev):
            for w in workers:
                line.wait_stream(w.s)
            line.wait_stream(side)
            r1.record(line)
        r1.synchronize()
        round_ms += r0.elapsed_time(r1)
    torch.cuda.synchronize()
    wall = round_ms / rounds   # device time of a round (master GPU's timeline)
    center = C_host if variant in ("orig", "orig_overlap", "sync1") else master.C[:n].cpu().numpy()
    return {c: v / rounds for c, v in cat.items()}, wall, eval_fn(center)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=min(4, torch.cuda.device_count()))
    ap.add_argument("--rounds", type=int, default=200)
    ap.add_argument("--model", default="lenet")
    ap.add_argument("--budget-scale", type=float, default=1.0)
    a = ap.parse_args()
    spec = network.MODELS[a.model](seed=0)
    from paper_1708_02983_b200.network import view_table
    LAYERS.extend((v.offset, v.offset + v.size) for v in view_table(spec))
    tr = normalize(gen_synthetic(10, spec.input_dim, 6000, seed=0, separation=5.0))
    te = normalize(gen_synthetic(10, spec.input_dim, 100, seed=1, separation=5.0))
    prob = NetworkProblem(spec, tr, te)
    ds = (np.ascontiguousarray(tr.samples, dtype=np.float32), tr.labels.astype(np.int32))
    hy = HyperParams(eta=0.05, rho=0.25)
    init = np.asarray(prob.init_weights(), dtype=np.float32)
    rows = []
    budgets = {"orig": 5000, "orig_overlap": 5000, "sync1": 1000, "sync2": 1000, "sync3": 1000}
    names = {"orig": "Original EASGD* (host master, per-layer msgs)",
             "orig_overlap": "Original EASGD (host master, per-layer msgs, overlap)",
             "sync1": "Sync EASGD1 (host master)", "sync2": "Sync EASGD2 (GPU master, peer copies)",
             "sync3": "Sync EASGD3 (GPU master, overlapped)"}
    serial_of = {"orig_overlap": "orig", "sync3": "sync2"}
    meas = {}
    for v in ("orig", "orig_overlap", "sync1", "sync2", "sync3"):
        workers = [Worker(i, torch.device("cuda", i % a.gpus), prob, init, 64, 3, ds) for i in range(a.gpus)]
        overlap = v in serial_of
        run(v, workers, hy, 10, overlap, lambda c: 0.0)   # warm-up (graphs, kernels)
        cat, round_ms, _ = run(v, workers, hy, a.rounds, overlap, lambda c: 0.0)
        meas[v] = (cat, round_ms)
        serial = sum(cat.values())
        comm = sum(cat[c] for c in COMM)
        if overlap:   # exposed comm = overlapped round - (its serial twin's round - its comm)
            cat0, round0 = meas[serial_of[v]]
            exposed = max(0.0, round_ms - (round0 - sum(cat0[c] for c in COMM)))
        else:
            exposed = comm
        iters = int(budgets[v] * a.budget_scale)
        rows.append({"method": names[v], "iterations": iters, "ms_per_iter": round_ms,
                     "time_s": round_ms * iters / 1e3, "shares": {c: cat[c] / serial for c in CATS}, "ms": cat,
                     "comm_ms": comm, "exposed_comm_ms": exposed, "comm_ratio": min(1.0, exposed / round_ms)})
        print(json.dumps(rows[-1]), flush=True)
    print("\n| method | iterations | time | ms/iter | " + " | ".join(CATS) + " | comm ratio |")
    print("|---|---:|---:|---:|" + "---:|" * len(CATS) + "---:|")
    for r in rows:
        print(f"| {r['method']} | {r['iterations']} | {r['time_s']:.2f} s | {r['ms_per_iter']:.3f} | " +
              " | ".join(f"{100 * r['shares'][c]:.0f}%" for c in CATS) + f" | {100 * r['comm_ratio']:.0f}% |")


if __name__ == "__main__":
    main()
