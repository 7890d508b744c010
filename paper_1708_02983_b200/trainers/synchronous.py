"""Bulk-synchronous elastic averaging on the device — the north-star path
(reference trainers/synchronous.py:47-219).

Per round, exactly the reference's arithmetic (``_sync_round``, :57-64):
every worker i computes g_i at W_i(t); S = sum_i W_i(t) (pre-update);
W_i(t+1) = (W_i - eta g_i) - eta rho (W_i - C_t); C(t+1) = C_t + eta rho (S - P C_t).

B200 mapping:
* one process per GPU (torchrun); each process holds P/world worker replicas
  as rows of one (nrep, ldw) fp32 tensor plus a replica of the center;
* S = local fixed-order replica sum (the reference's binomial order, exact
  when all workers are local) + one NCCL allreduce of the packed buffer over
  NVLink/NVSwitch (replaces tree_sum / Alg. 3's broadcast+reduce);
* the worker steps of all local replicas and the center step are one fused
  HBM-streaming kernel (esgd_sync_update_f32), every rank updating its own
  identical center replica;
* ``sync-easgd3``: the sum+allreduce runs on a side stream concurrently with
  the round's forward/backward (both only read W(t)); 1 and 2
  serialize it. Placement differences between easgd1/2 are pricing-only in
  the reference (:1-28) and arithmetic-identical here as there;
* the round (sampling, forward/backward, sum, allreduce, update) is captured
  once in a CUDA graph and replayed, so the host cost per round is one launch.
"""

from __future__ import annotations

import os
import time
import warnings

import numpy as np
import torch
import torch.distributed as dist

from .. import _lib
from ..device import require_cuda, round_up, stream_ptr
from ..errors import InputError
from ..fabric.collectives import CabiComm, allreduce_sum_, local_workers, replica_sum_, world
from ..fabric.nvls import NvlsRound, nvls_fused_single_kernel, nvls_reserve_sms, nvls_wanted
from ..fabric.engine import CATEGORIES
from ..rng import stream_seed
from ..updates import sync_update_, sync_update_solo_, sync_update_sum_
from .common import Recorder
from .config import TrainerConfig
from .records import RunRecord

SYNC_METHODS = ("sync-easgd1", "sync-easgd2", "sync-easgd3", "group-easgd")


class SyncEngine:
    """Device state and one-round step of a Sync-EASGD run on this rank."""

    def __init__(self, cfg: TrainerConfig, problem, use_graph: bool = True, use_tc: bool = True,
                 profile_rounds: int = 2):
        if cfg.method not in SYNC_METHODS:
            raise InputError(f"not a bulk-synchronous method: {cfg.method}")
        self.cfg, self.problem = cfg, problem
        self.P = cfg.cluster.workers
        self.world, self.rank = world()
        mine = local_workers(self.P, self.world, self.rank)
        self.nrep = len(mine)
        self.first = mine.start
        self.groups = cfg.cluster.groups if cfg.method == "group-easgd" else 1
        if self.groups > 1 and self.world > 1 and (self.nrep % (self.P // self.groups)) and \
                ((self.P // self.groups) % self.nrep):
            raise InputError("group-easgd across processes needs groups aligned to ranks")
        self.device = require_cuda()
        self.overlap = cfg.method == "sync-easgd3"
        init = np.asarray(problem.init_weights(), dtype=np.float32).reshape(-1)
        self.n = n = init.size
        self.ldw = ld = round_up(n, 64)
        dev = self.device
        self.W = torch.zeros((self.nrep, ld), dtype=torch.float32, device=dev)
        self.W[:, :n] = torch.from_numpy(init).to(dev)
        self.G = torch.zeros_like(self.W)
        self.C = torch.zeros(ld, dtype=torch.float32, device=dev)
        self.C[:n] = self.W[0, :n]
        self.S = torch.zeros(ld, dtype=torch.float32, device=dev)
        gsize = self.P // self.groups
        self.local_groups = max(1, self.nrep // gsize) if self.groups > 1 else 1
        self.partials = (torch.zeros((self.local_groups, ld), dtype=torch.float32, device=dev)
                         if self.local_groups > 1 else None)
        # without groups the update kernel also forms the next round's local
        # replica sum (esgd_sync_update_sum_f32), so S holds sum_r W_r at the
        # start of every round and the round only allreduces it
        self.fused_sum = self.groups == 1 and self.nrep <= 8
        # one worker in total: the sum is W(t) itself; the update reads W, G, C
        # and writes W, C (esgd_sync_update_solo_f32, 20 instead of 28 B/param)
        self.solo = self.P == 1 and self.world == 1
        if self.fused_sum and not self.solo:
            replica_sum_(self.S, self.W, self.n)
        # multi-GPU: the round's collective + update as ONE kernel over NVLink
        # SHARP multicast (fabric/nvls.py, csrc/nvls.cu) when the fabric has it;
        # otherwise one NCCL allreduce of S per round
        self.nvls, self.parity = None, 0
        self.plan = problem.bind(dev, self.nrep, cfg.batch_size, ld, use_tc=use_tc)
        self.plan.set_streams([stream_seed(cfg.seed, w) for w in range(self.first, self.first + self.nrep)])
        self.comm = torch.cuda.Stream(device=dev)
        self.use_graph = use_graph
        self.graph = None
        self.profile_rounds = profile_rounds
        self.phase_ms = {c: 0.0 for c in CATEGORIES}
        self.profiled = 0
        if self.world > 1:  # bring NCCL up outside any capture
            allreduce_sum_(torch.zeros(1, device=dev))
            torch.cuda.synchronize()
            if self.fused_sum and nvls_wanted():
                try:
                    self.nvls = NvlsRound(ld, dev, nrep=self.nrep)
                except Exception as exc:  # no multicast object support: NCCL path
                    warnings.warn(f"NVLS multicast unavailable ({exc}); using one NCCL allreduce per round",
                                  RuntimeWarning, stacklevel=2)
                    self.nvls = None
                    torch.cuda.synchronize()
            if self.nvls is not None:
                self.nvls.C[0].copy_(self.C)
                self.nvls.S[0].copy_(self.S)
                self.C, self.S = self.nvls.C[0], self.nvls.S[0]
                if self.nvls.w_src:  # peers read this rank's W in place
                    self.nvls.W.copy_(self.W)
                    self.W = self.nvls.W
                torch.cuda.synchronize()
        # ESGD_COLLECTIVE=cabi: the allreduce through libesgd's own NCCL
        # communicator (the C-ABI path of hosts without torch.distributed)
        self.cabi = None
        if self.world > 1 and self.nvls is None and os.environ.get("ESGD_COLLECTIVE") == "cabi":
            self.cabi = CabiComm(dev)
            torch.cuda.synchronize()
        self.graphs = [None, None]
        self._nocomm = False
        self.nvls_single = nvls_fused_single_kernel()
        self.collective = (("nvls-ce" if self.nvls.ce else "nvls-fused") if self.nvls is not None else
                           ("nccl-cabi" if self.cabi is not None else
                            ("nccl-allreduce" if self.world > 1 else "none")))

    # ---- one round ------------------------------------------------------------
    def _sum(self, stream) -> None:
        if self.solo or self._nocomm:
            return
        if self.nvls is not None:
            if not self.nvls_single:  # center slice over NVLS, overlapped with the backward
                self.nvls.center(self.parity, self.P, self.cfg.hyper, stream)
            return
        if self.fused_sum:  # local sum already formed by the previous update
            self._allreduce(stream)
            return
        if self.partials is not None:
            gsize = self.nrep // self.local_groups
            for g in range(self.local_groups):
                replica_sum_(self.partials[g], self.W[g * gsize:(g + 1) * gsize], self.n, stream)
            replica_sum_(self.S, self.partials, self.n, stream)
        else:
            replica_sum_(self.S, self.W, self.n, stream)
        self._allreduce(stream)

    def _allreduce(self, stream) -> None:
        if self.cabi is not None:
            self.cabi.allreduce_sum_(self.S, stream)
        else:
            allreduce_sum_(self.S)  # torch.distributed, on the current stream

    def _gradient(self, stream) -> None:
        # NVLS overlap: the center kernel takes `reserve` whole SMs, the
        # forward/backward's persistent GEMMs the others (their grids are
        # fixed at launch / graph capture; results do not depend on them)
        reserve = (nvls_reserve_sms() if self.nvls is not None and self.overlap and not self.nvls_single
                   and not self._nocomm and not self.solo else 0)
        if reserve:
            _lib.call("esgd_set_sm_reserve", reserve)
        try:
            self.plan.gradient(self.G, self.W, stream_ptr(stream))
        finally:
            if reserve:
                _lib.call("esgd_set_sm_reserve", 0)

    def _update(self, stream) -> None:
        if self._nocomm:  # timing twin without the cross-GPU part: the local fused update only
            if self.nvls is not None and self.nvls.w_src:
                self.nvls.workers(self.W, self.G, self.parity, self.cfg.hyper, stream)
            elif self.solo:
                sync_update_solo_(self.W, self.G, self.C, self.n, self.cfg.hyper, stream)
            else:
                sync_update_sum_(self.W, self.G, self.C, self.S, self.S, self.n, self.P, self.cfg.hyper, stream)
            return
        if self.nvls is not None:
            if self.nvls_single:
                self.nvls.update(self.W, self.G, self.parity, self.P, self.cfg.hyper, stream)
            else:
                self.nvls.workers(self.W, self.G, self.parity, self.cfg.hyper, stream)
        elif self.solo:
            sync_update_solo_(self.W, self.G, self.C, self.n, self.cfg.hyper, stream)
        elif self.fused_sum:
            sync_update_sum_(self.W, self.G, self.C, self.S, self.S, self.n, self.P, self.cfg.hyper, stream)
        else:
            sync_update_(self.W, self.G, self.C, self.S, self.n, self.P, self.cfg.hyper, stream)

    def step_eager(self, ev: dict | None = None) -> None:
        cs = torch.cuda.current_stream()
        rec = (lambda k, s: ev[k].record(s)) if ev is not None else (lambda k, s: None)
        rec("t0", cs)
        if self.overlap:
            self.comm.wait_stream(cs)
            with torch.cuda.stream(self.comm):
                rec("c0", self.comm)
                self._sum(self.comm)
                rec("c1", self.comm)
            self._gradient(cs)
            rec("g1", cs)
            cs.wait_stream(self.comm)
        else:
            self._gradient(cs)
            rec("g1", cs)
            rec("c0", cs)
            self._sum(cs)
            rec("c1", cs)
        rec("j", cs)
        self._update(cs)
        rec("u1", cs)

    def _capture(self) -> None:
        g = torch.cuda.CUDAGraph()
        # capture on a side stream (torch requirement); the graph then replays anywhere
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        rng_before = self.plan.rng.state.clone() if hasattr(self.plan, "rng") else None
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self.step_eager()
        torch.cuda.current_stream().wait_stream(s)
        if rng_before is not None:  # capture does not execute, but keep state untouched
            self.plan.rng.state.copy_(rng_before)
        if self.nvls is not None:
            self.graphs[self.parity] = g
        else:
            self.graphs = [g, g]
        self.graph = g

    def exposed_comm(self, rounds: int = 10) -> dict:
        """Exposed communication of the graph-replayed round, measured: the
        device time of `rounds` replays of the captured round minus that of a
        captured twin with the cross-GPU part removed (no allreduce / NVLS
        center; the local fused update instead), max over ranks. This is the
        part of the round the collective adds after overlap (the reference's
        exposed-interval accounting, fabric/engine.py:87-115). Timing only:
        the twin's rounds leave the ranks' centers inconsistent, so call it
        after the run's real rounds."""
        def timed(graph):
            torch.cuda.synchronize()
            if self.world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(rounds):
                graph.replay()
            b.record()
            b.synchronize()
            return _max_over_ranks(a.elapsed_time(b) / 1e3 / rounds, self.device)

        full = self.graphs[self.parity]
        if full is None:
            self._capture()
            full = self.graphs[self.parity]
        t_full = timed(full)
        saved = (self.graph, list(self.graphs))
        self._nocomm = True
        try:
            self._capture()
            twin = self.graphs[self.parity]
        finally:
            self._nocomm = False
            self.graph, self.graphs = saved
        t_local = timed(twin)
        exposed = max(0.0, t_full - t_local)
        return {"round_s": t_full, "round_without_comm_s": t_local, "exposed_s": exposed,
                "fraction": exposed / t_full if t_full > 0 else 0.0, "rounds": rounds,
                "collective": self.collective}

    def time_collective(self, reps: int = 10) -> dict:
        """The round's cross-GPU part alone (no overlapping work): the NCCL
        allreduce of the packed local sum S, or the NVLS center kernel
        (barrier + multimem ld_reduce of this rank's slice of S + center step +
        multimem store), `reps` eager launches between barriers, max over ranks.
        Per GPU the NVLS kernel moves (N-1)/N * 4|W| B in (the switch-reduced
        slice) and the same out (its broadcast), like a ring allreduce's
        2 (N-1)/N * 4|W|. Timing only (rewrites S / the next center)."""
        if self.world < 2:
            return {"s": 0.0, "bytes_per_gpu": 0, "GBps": None}
        cs = torch.cuda.current_stream()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            if self.nvls is not None:
                self.nvls.center(self.parity, self.P, self.cfg.hyper, cs)
            else:
                self._allreduce(cs)
        b.record()
        b.synchronize()
        t = _max_over_ranks(a.elapsed_time(b) / 1e3 / reps, self.device)
        nbytes = 2.0 * (self.world - 1) / self.world * 4 * self.ldw
        return {"s": t, "bytes_per_gpu": nbytes, "GBps": nbytes / t / 1e9 if t > 0 else None,
                "collective": self.collective}

    def close(self) -> None:
        """Release the captured rounds and the C-ABI communicator (if any).
        Idempotent; the engine cannot step afterwards."""
        if self.cabi is not None:
            self.graph, self.graphs = None, [None, None]  # graphs hold work on the communicator
            torch.cuda.synchronize(self.device)
            self.cabi.close()
            self.cabi = None

    def after_external_write(self) -> None:
        """W / C were overwritten outside the round (resume): re-form the local
        replica sum the fused update path keeps in S."""
        if self.fused_sum and not self.solo:
            replica_sum_(self.S, self.W, self.n)
        torch.cuda.synchronize()

    def advance(self) -> None:
        """After a round: the NVLS path double-buffers S/C by round parity."""
        if self.nvls is not None:
            self.parity ^= 1
            self.C, self.S = self.nvls.C[self.parity], self.nvls.S[self.parity]

    def step(self) -> None:
        """Enqueue one round (graph replay once captured; the NVLS path keeps
        one graph per round parity)."""
        k = self.parity
        if self.graphs[k] is not None:
            self.graphs[k].replay()
            self.advance()
            return
        if self.use_graph and self.profiled >= self.profile_rounds:
            try:
                self._capture()
            except Exception as exc:  # capture unsupported here: stay eager
                warnings.warn(f"CUDA graph capture of the round failed ({exc}); running eagerly",
                              RuntimeWarning, stacklevel=2)
                self.use_graph = False
                torch.cuda.synchronize()
            if self.graphs[k] is not None:
                self.graphs[k].replay()
                self.advance()
                return
        if self.profiled < self.profile_rounds:
            self._profiled_step()
        else:
            self.step_eager()
        self.advance()

    def _profiled_step(self) -> None:
        names = ("t0", "c0", "c1", "g1", "j", "u1")
        ev = {k: torch.cuda.Event(enable_timing=True) for k in names}
        self.step_eager(ev)
        ev["u1"].synchronize()
        fb = ev["t0"].elapsed_time(ev["g1"])
        if self.overlap:
            exposed = max(0.0, ev["g1"].elapsed_time(ev["j"]))
        else:
            exposed = ev["c0"].elapsed_time(ev["c1"])
        self.phase_ms["forward_backward"] += fb
        self.phase_ms["peer_param"] += exposed
        self.phase_ms["worker_update"] += ev["j"].elapsed_time(ev["u1"])
        self.profiled += 1

    # ---- results --------------------------------------------------------------
    def center_host(self) -> np.ndarray:
        return self.C[:self.n].cpu().numpy()

    def workers_host(self) -> list[np.ndarray]:
        local = self.W[:, :self.n].contiguous()
        if self.world > 1:
            bufs = [torch.empty_like(local) for _ in range(self.world)]
            dist.all_gather(bufs, local)
            local = torch.cat(bufs)
        return [local[i].cpu().numpy() for i in range(self.P)]

    def breakdown(self, total_s: float) -> dict[str, float]:
        out = {c: 0.0 for c in CATEGORIES}
        if self.profiled:
            per_round = {k: v / self.profiled / 1e3 for k, v in self.phase_ms.items()}
            tot = sum(per_round.values())
            scale = total_s / (tot * self.cfg.iterations) if tot > 0 else 0.0
            for k, v in per_round.items():
                out[k] = v * self.cfg.iterations * scale
        return out


def _max_over_ranks(x: float, device) -> float:
    if world()[0] > 1:
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return x


def run_synchronous(cfg: TrainerConfig, problem, cm=None, **engine_kw) -> RunRecord:
    eng = SyncEngine(cfg, problem, **engine_kw)
    try:
        return _run_rounds(eng, cfg, problem)
    finally:
        eng.close()


def _run_rounds(eng, cfg: TrainerConfig, problem) -> RunRecord:
    rec = Recorder(problem, cfg.eval_every, cfg.iterations)
    elapsed = 0.0
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    for t in range(cfg.iterations):
        eng.step()
        if rec.due(t + 1):
            t1.record()
            t1.synchronize()
            elapsed += t0.elapsed_time(t1) / 1e3
            rec.record(t + 1, _max_over_ranks(elapsed, eng.device), eng.C[:eng.n])
            t0.record()
    total = _max_over_ranks(elapsed, eng.device)
    info = {"engine": "cuda", "world": eng.world, "replicas_per_rank": eng.nrep,
            "graph": eng.graph is not None, "overlap": eng.overlap, "collective": eng.collective}
    return rec.build(cfg.method, total, eng.center_host(), breakdown=eng.breakdown(total),
                     worker_weights=eng.workers_host(), engine_info=info)
