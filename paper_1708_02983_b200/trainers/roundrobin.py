"""Original EASGD (Alg. 1; reference trainers/roundrobin.py:32-132) on the
device: one worker per round in strict round-robin order; its worker step
against the center and the incremental center step with its pre-update
weights are one fused kernel (esgd_exchange_update_f32). The paper's slow
baseline, kept for the Table-3 comparison; deterministic and bitwise equal
to the fp32 reference arithmetic."""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib
from ..device import require_cuda, stream_ptr
from ..errors import InputError
from ..fabric.engine import CATEGORIES
from ._slots import WorkerSlot
from .common import Recorder
from .config import TrainerConfig
from .records import RunRecord


def run_original_easgd(cfg: TrainerConfig, problem, cm=None) -> RunRecord:
    if cfg.method != "original-easgd":
        raise InputError(f"not the round-robin method: {cfg.method}")
    dev = require_cuda()
    G = cfg.cluster.workers
    h = cfg.hyper
    init = np.asarray(problem.init_weights(), dtype=np.float32).reshape(-1)
    n = init.size
    slots = [WorkerSlot(w, problem, init, dev, cfg.batch_size, cfg.seed, momentum=False, snapshot=False)
             for w in range(G)]
    C = torch.zeros(slots[0].ld, dtype=torch.float32, device=dev)
    C[:n] = torch.from_numpy(init).to(dev)
    lib = _lib.load()
    rec = Recorder(problem, cfg.eval_every, cfg.iterations)
    s = stream_ptr()
    elapsed = 0.0
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # measured breakdown (reference categories, fabric/engine.py): per round a
    # gradient (forward_backward) and the fused exchange kernel, which is both
    # the worker step and the center's incremental step (worker_update /
    # master_update, split evenly); no message leaves the device
    marks = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
              torch.cuda.Event(enable_timing=True)) for _ in range(cfg.iterations)]
    torch.cuda.synchronize()
    t0.record()
    for t in range(cfg.iterations):
        sl = slots[t % G]
        e = marks[t]
        e[0].record()
        sl.plan.gradient(sl.G, sl.W, s)
        e[1].record()
        _lib.check(lib.esgd_exchange_update_f32(sl.W.data_ptr(), sl.G.data_ptr(), C.data_ptr(), n,
                                                h.eta32, h.etarho32, s))
        e[2].record()
        if rec.due(t + 1):
            t1.record()
            t1.synchronize()
            elapsed += t0.elapsed_time(t1) / 1e3
            rec.record(t + 1, elapsed, C[:n])
            t0.record()
    torch.cuda.synchronize()
    bd = {c: 0.0 for c in CATEGORIES}
    fb = sum(e[0].elapsed_time(e[1]) for e in marks) / 1e3
    ex = sum(e[1].elapsed_time(e[2]) for e in marks) / 1e3
    bd["forward_backward"] = fb
    bd["worker_update"] = bd["master_update"] = ex / 2
    return rec.build(cfg.method, elapsed, C[:n].cpu().numpy(), breakdown=bd,
                     worker_weights=[sl.W[0, :n].cpu().numpy() for sl in slots],
                     engine_info={"engine": "cuda"})
