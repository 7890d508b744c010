"""Parameter-server schedules on the device (reference
trainers/asynchronous.py:46-264): workers run free on their own CUDA streams
(spread over the visible GPUs of this process); a master stream on device 0
owns the center and serves exchanges strictly first-come-first-served.

FCFS is real, not simulated: a worker's request "arrives" when its previous
update has completed on the device; the host scheduler polls those
completion events and enqueues each exchange on the master stream in the
order it observes them (ties in one polling sweep by worker id, as the
reference's FcfsQueue, fabric/engine.py:125-148). The master stream is the
sole writer of the center — the whole-buffer mutual exclusion of the locked
modes (:190-192) — and every exchange is two kernels on it.

* async-easgd / async-measgd: the worker ships W (no dependency on its
  gradient, which overlaps the round trip); the master replies with the
  pre-update center (a device copy into the worker's snapshot) and folds W
  in with easgd_center_incremental; the worker then applies the elastic
  (momentum) step against that snapshot (:121-142).
* async-sgd / async-msgd: the worker ships its gradient; the master applies
  (momentum) SGD to the center and the worker adopts the new center.

Device master (default for async-easgd / async-measgd without periodic
evaluation, ``ESGD_ASYNC_MASTER=device``): no host in the loop at all — the
master is one persistent kernel on device 0 serving tickets FCFS, each worker
stream runs post -> gradient -> wait -> elastic step (csrc/async.cu). The
host only enqueues the workers' cycles in bounded chunks. With periodic
evaluation (eval_every > 0) or ``ESGD_ASYNC_MASTER=host`` the host-polled
master above runs instead.
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from .. import _lib
from ..device import require_cuda, stream_ptr
from ..errors import InputError
from ..fabric.engine import CATEGORIES
from ._slots import WorkerSlot, split_iterations, worker_devices
from .common import Recorder
from .config import TrainerConfig
from .records import RunRecord

ASYNC_METHODS = ("async-sgd", "async-easgd", "async-msgd", "async-measgd")
_EXCHANGES_WEIGHTS = {"async-easgd": False, "async-measgd": True}
_PUSHES_GRADIENT = {"async-sgd": False, "async-msgd": True}


def run_asynchronous(cfg: TrainerConfig, problem, cm=None, devices=None) -> RunRecord:
    if cfg.method not in ASYNC_METHODS:
        raise InputError(f"not a parameter-server method: {cfg.method}")
    master_dev = require_cuda()
    P = cfg.cluster.workers
    h = cfg.hyper
    eta, mu, er = h.eta32, h.mu32, h.etarho32
    weights_mode = cfg.method in _EXCHANGES_WEIGHTS
    momentum = _EXCHANGES_WEIGHTS.get(cfg.method) or _PUSHES_GRADIENT.get(cfg.method)
    quotas = split_iterations(cfg.iterations, P)
    init = np.asarray(problem.init_weights(), dtype=np.float32).reshape(-1)
    n = init.size
    devs = devices or worker_devices(P)
    slots = [WorkerSlot(w, problem, init, devs[w], cfg.batch_size, cfg.seed,
                        momentum=bool(momentum) and weights_mode, snapshot=weights_mode) for w in range(P)]
    if weights_mode and cfg.eval_every == 0 and os.environ.get("ESGD_ASYNC_MASTER", "device") == "device":
        for sl in slots:
            sl.prepare_graph()
        if all(sl.graph is not None for sl in slots):  # (eager gradients could lazily load kernels mid-run)
            return _run_device_master(cfg, problem, slots, quotas, master_dev, bool(momentum))
    ld = slots[0].ld
    C = torch.zeros(ld, dtype=torch.float32, device=master_dev)
    C[:n] = torch.from_numpy(init).to(master_dev)
    Vm = torch.zeros_like(C) if (momentum and not weights_mode) else None
    master = torch.cuda.Stream(device=master_dev)
    ms = stream_ptr(master)
    staging = {w: torch.zeros(ld, dtype=torch.float32, device=master_dev)
               for w in range(P) if slots[w].device != master_dev}
    lib = _lib.load()
    rec = Recorder(problem, cfg.eval_every, cfg.iterations)

    ready: list[torch.cuda.Event | None] = [None] * P   # request arrival events
    grad_busy = [0.0] * P
    master_busy = 0.0

    def enqueue_cycle(w: int):
        """Worker w's gradient for its next cycle (+ gradient-push request)."""
        sl = slots[w]
        with torch.cuda.device(sl.device), torch.cuda.stream(sl.stream):
            sl.gradient()
            if not weights_mode:
                ev = torch.cuda.Event()
                ev.record(sl.stream)
                ready[w] = ev

    def serve(w: int):
        """Master serves worker w's exchange (FCFS position decided by caller)."""
        sl = slots[w]
        ev = ready[w]
        with torch.cuda.device(master_dev), torch.cuda.stream(master):
            if ev is not None:
                master.wait_event(ev)
            if weights_mode:
                src = sl.w()
                if w in staging:
                    staging[w][:n].copy_(src, non_blocking=True)
                    src = staging[w][:n]
                # reply the pre-update center, then fold the worker's weights in
                sl.snap[:n].copy_(C[:n], non_blocking=True)
                _lib.check(lib.esgd_center_incr_f32(C.data_ptr(), C.data_ptr(), src.data_ptr(), n, er, ms))
            else:
                g = sl.G[0, :n]
                if w in staging:
                    staging[w][:n].copy_(g, non_blocking=True)
                    g = staging[w][:n]
                if momentum:
                    _lib.check(lib.esgd_msgd_step_f32(C.data_ptr(), Vm.data_ptr(), g.data_ptr(), n, eta, mu, ms))
                else:
                    _lib.check(lib.esgd_sgd_step_f32(C.data_ptr(), g.data_ptr(), n, eta, ms))
                sl.W[0, :n].copy_(C[:n], non_blocking=True)
            done_ev = torch.cuda.Event()
            done_ev.record(master)
        with torch.cuda.device(sl.device), torch.cuda.stream(sl.stream):
            sl.stream.wait_event(done_ev)
            if weights_mode:
                if momentum:
                    _lib.check(lib.esgd_measgd_update_f32(sl.W.data_ptr(), sl.V.data_ptr(), sl.G.data_ptr(),
                                                          sl.snap.data_ptr(), n, eta, mu, er, sl.s))
                else:
                    _lib.check(lib.esgd_worker_step_f32(sl.W.data_ptr(), sl.W.data_ptr(), sl.G.data_ptr(),
                                                        sl.snap.data_ptr(), n, eta, er, sl.s))
                nxt = torch.cuda.Event()
                nxt.record(sl.stream)
                ready[w] = nxt
        sl.done += 1
        if sl.done < quotas[w]:
            enqueue_cycle(w)

    torch.cuda.synchronize()
    t_start = time.perf_counter()
    paused = 0.0
    for w in range(P):
        if quotas[w] > 0:
            enqueue_cycle(w)
    services = 0
    waiting = [w for w in range(P) if quotas[w] > 0]
    while waiting:
        arrived = [w for w in waiting if ready[w] is None or ready[w].query()]
        if not arrived:
            time.sleep(0)
            continue
        for w in arrived:  # one polling sweep: ties by worker id
            serve(w)
            services += 1
            if rec.due(services):
                master.synchronize()  # the queued exchanges up to here are run time, not eval time
                p0 = time.perf_counter()
                rec.record(services, p0 - t_start - paused, C[:n])
                paused += time.perf_counter() - p0
        waiting = [w for w in range(P) if slots[w].done < quotas[w]]
    torch.cuda.synchronize()
    total = time.perf_counter() - t_start - paused
    info = {"engine": "cuda", "devices": sorted({str(d) for d in devs}), "fcfs": "host-polled completion order"}
    bd = {c: 0.0 for c in CATEGORIES}
    return rec.build(cfg.method, total, C[:n].cpu().numpy(), breakdown=bd,
                     worker_weights=[sl.W[0, :n].cpu().numpy() for sl in slots], engine_info=info)


def _run_device_master(cfg: TrainerConfig, problem, slots, quotas, master_dev, momentum: bool) -> RunRecord:
    """async-easgd / async-measgd with the master as one persistent kernel
    (esgd_async_master_f32, FCFS by ticket) and every worker cycle enqueued on
    the worker's own stream: post -> gradient -> wait -> elastic step."""
    lib = _lib.load()
    P = len(slots)
    n, ld = slots[0].n, slots[0].ld
    h = cfg.hyper
    eta, mu, er = h.eta32, h.mu32, h.etarho32
    init = slots[0].W[0, :n].to(master_dev)
    C = torch.zeros(ld, dtype=torch.float32, device=master_dev)
    C[:n] = init
    mi = master_dev.index if master_dev.index is not None else 0
    for sl in slots:
        di = sl.device.index if sl.device.index is not None else 0
        if di != mi:
            _lib.check(lib.esgd_enable_peer_access(di, mi), "peer access")
            _lib.check(lib.esgd_enable_peer_access(mi, di), "peer access")
    ctl = torch.zeros(lib.esgd_async_ctl_ints(P), dtype=torch.int32, device=master_dev)
    wptr = torch.tensor([sl.W.data_ptr() for sl in slots], dtype=torch.int64, device=master_dev)
    sptr = torch.tensor([sl.snap.data_ptr() for sl in slots], dtype=torch.int64, device=master_dev)
    posts = [torch.zeros(1, dtype=torch.int32, device=sl.device) for sl in slots]
    services = int(sum(quotas))
    master = torch.cuda.Stream(device=master_dev)
    chunk = int(os.environ.get("ESGD_ASYNC_CHUNK", "32"))
    for sl in slots:  # graph capture synchronises the device: before the master runs
        sl.prepare_graph()
    # every kernel a worker cycle launches must be loaded before the master
    # spins (lazy loading at a first launch can wait on running kernels)
    for d in {sl.device for sl in slots} | {master_dev}:
        with torch.cuda.device(d):
            _lib.check(lib.esgd_async_preload(), "async preload")
            z = torch.zeros(4, device=d)
            if momentum:
                _lib.check(lib.esgd_measgd_update_f32(z.data_ptr(), z.data_ptr(), z.data_ptr(), z.data_ptr(), 4,
                                                      eta, mu, er, None))
            else:
                _lib.check(lib.esgd_worker_step_f32(z.data_ptr(), z.data_ptr(), z.data_ptr(), z.data_ptr(), 4,
                                                    eta, er, None))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t_start = time.perf_counter()
    with torch.cuda.device(master_dev):
        t0.record(master)
    _lib.check(lib.esgd_async_master_f32(C.data_ptr(), n, wptr.data_ptr(), sptr.data_ptr(), ctl.data_ptr(), P,
                                         services, er, int(os.environ.get("ESGD_ASYNC_CTAS", "8")),
                                         stream_ptr(master)), "async master")

    def cycle(w: int) -> None:
        sl = slots[w]
        with torch.cuda.device(sl.device), torch.cuda.stream(sl.stream):
            _lib.check(lib.esgd_async_post(ctl.data_ptr(), P, w, posts[w].data_ptr(), sl.s), "async post")
            sl.gradient()
            _lib.check(lib.esgd_async_wait(ctl.data_ptr(), P, w, posts[w].data_ptr(), sl.s), "async wait")
            if momentum:
                _lib.check(lib.esgd_measgd_update_f32(sl.W.data_ptr(), sl.V.data_ptr(), sl.G.data_ptr(),
                                                      sl.snap.data_ptr(), n, eta, mu, er, sl.s))
            else:
                _lib.check(lib.esgd_worker_step_f32(sl.W.data_ptr(), sl.W.data_ptr(), sl.G.data_ptr(),
                                                    sl.snap.data_ptr(), n, eta, er, sl.s))
        sl.done += 1

    # every worker's cycles are enqueued round-robin in chunks; a worker never
    # runs more than two chunks ahead of what has completed, so the host never
    # blocks on one full stream queue while another worker still needs its post
    marks: list[list[torch.cuda.Event]] = [[] for _ in range(P)]
    while any(sl.done < q for sl, q in zip(slots, quotas)):
        for w, sl in enumerate(slots):
            if sl.done >= quotas[w]:
                continue
            if len(marks[w]) >= 2:
                marks[w].pop(0).synchronize()
            for _ in range(min(chunk, quotas[w] - sl.done)):
                cycle(w)
            ev = torch.cuda.Event()
            ev.record(sl.stream)
            marks[w].append(ev)
    t1 = torch.cuda.Event(enable_timing=True)
    for sl in slots:
        with torch.cuda.device(master_dev):
            master.wait_stream(sl.stream)
    with torch.cuda.device(master_dev):
        t1.record(master)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_start
    err = int(ctl[1].item())
    if err:
        from ..errors import CudaError
        c = ctl.cpu().numpy()
        Q = 2 * P
        raise CudaError(f"async device master stalled (code {err}): tickets {c[0]}, published "
                        f"{c[16 + Q:16 + 2 * Q].tolist()}, served {c[16 + 2 * Q:16 + 2 * Q + P].tolist()}, "
                        f"posts {[int(x.item()) for x in posts]}, done {[sl.done for sl in slots]} of {quotas}")
    total = t0.elapsed_time(t1) / 1e3
    rec = Recorder(problem, 0, cfg.iterations)
    rec.record(cfg.iterations, total, C[:n])  # the final evaluation (off the clock)
    info = {"engine": "cuda", "devices": sorted({str(sl.device) for sl in slots}),
            "fcfs": "device tickets (persistent master kernel)", "wall_s": wall, "services": services}
    bd = {c: 0.0 for c in CATEGORIES}
    return rec.build(cfg.method, total, C[:n].cpu().numpy(), breakdown=bd,
                     worker_weights=[sl.W[0, :n].cpu().numpy() for sl in slots], engine_info=info)
