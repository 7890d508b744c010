"""Lock-free schedules on the device (reference trainers/hogwild.py:35-214):
every worker is its own CUDA stream (C4: many worker streams on one B200),
all racing on one shared center with no lock.

Per worker iteration (hogwild.py:175-183), all on the worker's stream:
  snap <- center            (device copy; a racing read, may mix generations)
  g    <- gradient(W)
  center += eta*rho*(W - snap)   (esgd_hogwild_apply_f32: vector red.global.add,
                                   element-granular, concurrent with the others)
  W    <- easgd_worker_step(W, g, snap)
hogwild-sgd: center += -eta*g ; W <- center (racing snapshot).
Convergence is statistical, as in the reference's threaded engine.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from .. import _lib
from ..device import require_cuda, stream_ptr
from ..errors import InputError
from ..fabric.engine import CATEGORIES
from ._slots import WorkerSlot, split_iterations
from .common import Recorder
from .config import TrainerConfig
from .records import RunRecord

HOGWILD_METHODS = ("hogwild-sgd", "hogwild-easgd")


def run_hogwild(cfg: TrainerConfig, problem, cm=None) -> RunRecord:
    if cfg.method not in HOGWILD_METHODS:
        raise InputError(f"not a lock-free method: {cfg.method}")
    dev = require_cuda()
    P = cfg.cluster.workers
    h = cfg.hyper
    eta, er = h.eta32, h.etarho32
    elastic = cfg.method == "hogwild-easgd"
    quotas = split_iterations(cfg.iterations, P)
    init = np.asarray(problem.init_weights(), dtype=np.float32).reshape(-1)
    n = init.size
    slots = [WorkerSlot(w, problem, init, dev, cfg.batch_size, cfg.seed, momentum=False, snapshot=elastic)
             for w in range(P)]
    C = torch.zeros(slots[0].ld, dtype=torch.float32, device=dev)
    C[:n] = torch.from_numpy(init).to(dev)
    lib = _lib.load()
    rec = Recorder(problem, cfg.eval_every, cfg.iterations)

    def body(sl: WorkerSlot, s: int, grad) -> None:
        """One lock-free iteration of worker sl on stream s (trainers/hogwild.py:175-183)."""
        if elastic:
            sl.snap[:n].copy_(C[:n], non_blocking=True)   # racy snapshot of the shared center
            grad()
            _lib.check(lib.esgd_hogwild_apply_f32(C.data_ptr(), sl.W.data_ptr(), sl.snap.data_ptr(), n, er, s))
            _lib.check(lib.esgd_worker_step_f32(sl.W.data_ptr(), sl.W.data_ptr(), sl.G.data_ptr(),
                                                sl.snap.data_ptr(), n, eta, er, s))
        else:
            grad()
            _lib.check(lib.esgd_hogwild_axpy_f32(C.data_ptr(), sl.G.data_ptr(), n, -eta, s))
            sl.W[0, :n].copy_(C[:n], non_blocking=True)

    graphs: dict[int, torch.cuda.CUDAGraph] = {}

    def iteration(sl: WorkerSlot):
        # first iteration eager (warm-up, lazy allocations), then the whole
        # iteration — snapshot, sampling, forward/backward, atomic center
        # update, worker step — replays as one CUDA graph on the worker's stream
        g = graphs.get(sl.wid)
        if g is None and sl.done >= 1:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(sl.stream)
            rng = getattr(sl.plan, "rng", None)
            before = rng.state.clone() if rng is not None else None
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                body(sl, stream_ptr(side), lambda: sl.plan.gradient(sl.G, sl.W, stream_ptr(side)))
            sl.stream.wait_stream(side)
            if before is not None:
                rng.state.copy_(before)
            graphs[sl.wid] = g
        with torch.cuda.stream(sl.stream):
            if g is not None:
                g.replay()
            else:
                body(sl, sl.s, sl.gradient)
        sl.done += 1

    torch.cuda.synchronize()
    t_start = time.perf_counter()
    paused = 0.0
    services = 0
    rnd = 0
    while services < cfg.iterations:
        for w, sl in enumerate(slots):  # round-robin issue; the streams then race freely
            if sl.done < quotas[w]:
                iteration(sl)
                services += 1
                if rec.due(services):
                    torch.cuda.synchronize()  # the queued work up to here is run time, not eval time
                    p0 = time.perf_counter()
                    rec.record(services, p0 - t_start - paused, C[:n])
                    paused += time.perf_counter() - p0
        rnd += 1
    torch.cuda.synchronize()
    total = time.perf_counter() - t_start - paused
    bd = {c: 0.0 for c in CATEGORIES}
    return rec.build(cfg.method, total, C[:n].cpu().numpy(), breakdown=bd,
                     worker_weights=[sl.W[0, :n].cpu().numpy() for sl in slots],
                     engine_info={"engine": "cuda", "streams": P, "lock": "none (vector red.global.add)"})
