"""Host-fed Sync-EASGD rounds: the dataset stays in pinned host memory and
every round's batch crosses PCIe, as with a data loader (the end-to-end
path `bench.py` reports as `e2e`). The default engine path (`run_trainer`)
keeps the training set resident in HBM instead.

* ``DmaFeed`` (ImageNet-sized rows): the workers' SplitMix64 streams draw the
  indices on the host; each drawn row is copied from the pinned dataset into
  one of two device batch buffers by DMA (``esgd_gather_rows_h2d``, a
  cudaMemcpyAsync per row run on a copy stream — no host gather, no SMs),
  overlapped with the previous round.
* ``ZeroCopyFeed`` (small rows): the round's sampling kernel draws the
  indices on the device and reads the rows straight from the pinned host
  dataset over PCIe (mapped pinned memory) inside the round's CUDA graph.

Both replay one CUDA graph per data buffer / round parity that also copies
the round's mean loss to pinned host memory; ``step()`` returns it.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _lib
from ..device import stream_ptr
from ..rng import CounterRng, stream_seed
from .synchronous import SyncEngine


class _GraphRounds:
    """One captured CUDA graph per round parity / data buffer: the round's
    sum (side stream), forward/backward, update and the D2H of its mean loss."""

    def _graph(self, k):
        if self.graphs[k] is None:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
                self._device_round(k)
            torch.cuda.current_stream().wait_stream(s)
            self.graphs[k] = g
        return self.graphs[k]


class DmaFeed(_GraphRounds):
    """Host data path for big rows (ImageNet-sized): the dataset lives in
    pinned host memory; each round's rows are drawn on the host with the
    workers' SplitMix64 streams and copied straight to one of two device
    batch buffers by DMA (esgd_gather_rows_h2d: one cudaMemcpyAsync per row
    on a copy stream — no host-side gather, no SMs), overlapped with the
    previous round; one CUDA graph per buffer runs the round and the D2H of
    the round's mean loss, which is read back after every round."""

    def __init__(self, prob, eng):
        self.prob, self.eng = prob, eng
        net = eng.plan.net
        self.net = net
        b, nrep, d = net.b, net.nrep, net.d_in
        X = np.ascontiguousarray(prob.train.samples, dtype=np.float32)
        self.n, self.d = X.shape
        self.Xp = torch.from_numpy(X).pin_memory()  # setup, outside the timed region
        self.Y = prob.train.labels.astype(np.int32)
        self.rngs = [CounterRng(stream_seed(eng.cfg.seed, w)) for w in range(eng.first, eng.first + nrep)]
        self.xb = [torch.empty((nrep, b * d), dtype=torch.float32, device="cuda") for _ in range(2)]
        self.yb = [torch.empty((nrep, b), dtype=torch.int32, device="cuda") for _ in range(2)]
        self.hy = [torch.empty((nrep, b), dtype=torch.int32).pin_memory() for _ in range(2)]
        self.loss = torch.empty(nrep, dtype=torch.float32).pin_memory()
        self.h2d_bytes = nrep * b * d * 4 + nrep * b * 4
        self.d2h_bytes = nrep * 4
        self.graphs = [None, None]
        self.copy = torch.cuda.Stream()
        self.ev = [torch.cuda.Event(), torch.cuda.Event()]
        self.x0, self.y0 = net.x, net.y
        self.cur = 0
        self._load(0)

    def _load(self, k):
        lib = _lib.load()
        net, hy = self.net, self.hy[k].numpy()
        for r, rng in enumerate(self.rngs):
            idx = np.ascontiguousarray(rng.randint_block(net.b, self.n), dtype=np.int64)
            hy[r] = self.Y[idx]
            _lib.check(lib.esgd_gather_rows_h2d(self.xb[k][r].data_ptr(), self.d * 4, self.Xp.data_ptr(),
                                                self.d * 4, idx.ctypes.data, net.b, self.d * 4, self.n,
                                                stream_ptr(self.copy)), "gather_rows_h2d")
        with torch.cuda.stream(self.copy):
            self.yb[k].copy_(self.hy[k], non_blocking=True)
        self.ev[k].record(self.copy)

    def _device_round(self, k):
        eng, net = self.eng, self.net
        cs = torch.cuda.current_stream()
        eng.comm.wait_stream(cs)
        with torch.cuda.stream(eng.comm):
            eng._sum(eng.comm)
        net.gradient(eng.G, eng.W, stream_ptr(cs))
        cs.wait_stream(eng.comm)
        eng._update(cs)
        self.loss.copy_(net.row_loss[:, :net.b].mean(dim=1), non_blocking=True)

    def _graph(self, k):
        # the round of buffer k reads xb[k] / yb[k] directly (captured pointers)
        self.net.x, self.net.y = self.xb[k], self.yb[k]
        try:
            return _GraphRounds._graph(self, k)
        finally:
            self.net.x, self.net.y = self.x0, self.y0

    def step(self):
        k = self.cur
        cs = torch.cuda.current_stream()
        cs.wait_event(self.ev[k])      # batch k on the device
        self._graph(k).replay()        # round + loss D2H (async)
        self.eng.advance()
        self._load(k ^ 1)              # next batch by DMA, concurrent with round k
        cs.synchronize()
        self.cur = k ^ 1
        return float(self.loss.numpy().mean())


class ZeroCopyFeed(_GraphRounds):
    """Host data path for small rows (MNIST-sized): the dataset lives in
    pinned host memory and the round's sampling kernel (esgd_sample_batch_f32,
    the workers' SplitMix64 streams on the device) reads the drawn rows
    straight from it over PCIe (mapped pinned memory) — each round's inputs
    cross host->device inside the round's CUDA graph, with no per-round host
    gather or copy call; the graph also does the D2H of the round's mean
    loss, which is read back after every round."""

    def __init__(self, prob, eng):
        self.prob, self.eng = prob, eng
        net = eng.plan.net
        self.net, self.plan = net, eng.plan
        b, nrep, d = net.b, net.nrep, net.d_in
        X = np.ascontiguousarray(prob.train.samples, dtype=np.float32)
        self.n, self.d = X.shape
        self.Xp = torch.from_numpy(X).pin_memory()
        self.Yp = torch.from_numpy(prob.train.labels.astype(np.int32)).pin_memory()
        self.loss = torch.empty(nrep, dtype=torch.float32).pin_memory()
        self.h2d_bytes = nrep * b * d * 4 + nrep * b * 4
        self.d2h_bytes = nrep * 4
        self.graphs = [None, None]

    def _device_round(self, k):
        eng, net, plan = self.eng, self.net, self.plan
        cs = torch.cuda.current_stream()
        _lib.check(_lib.load().esgd_sample_batch_f32(
            net.x.data_ptr(), net.x.stride(0), net.y.data_ptr(), None, self.Xp.data_ptr(), self.Yp.data_ptr(),
            self.n, self.d, plan.rng.state.data_ptr(), plan.rng.ticket.data_ptr(), net.b, net.nrep,
            stream_ptr(cs)), "sample_batch (pinned host rows)")
        eng.comm.wait_stream(cs)
        with torch.cuda.stream(eng.comm):
            eng._sum(eng.comm)
        net.gradient(eng.G, eng.W, stream_ptr(cs))
        cs.wait_stream(eng.comm)
        eng._update(cs)
        self.loss.copy_(net.row_loss[:, :net.b].mean(dim=1), non_blocking=True)

    def step(self):
        k = self.eng.parity if self.eng.nvls is not None else 0
        rng = self.plan.rng.state
        if self.graphs[k] is None:  # capture does not run the sampling kernel: keep the RNG as is
            before = rng.clone()
            self._graph(k)
            rng.copy_(before)
        self.graphs[k].replay()
        self.eng.advance()
        torch.cuda.current_stream().synchronize()
        return float(self.loss.numpy().mean())


class HostFedRun:
    """Sync-EASGD rounds of ``cfg`` on ``problem`` fed from host memory:
    ``step()`` runs one round (batch H2D inside) and returns its mean loss;
    ``h2d_bytes`` / ``d2h_bytes`` are the bytes each round moves; ``engine``
    is the underlying SyncEngine (center, workers)."""

    BIG_ROW_BYTES = 65536

    def __init__(self, cfg, problem):
        self.engine = SyncEngine(cfg, problem, use_graph=False, profile_rounds=0)
        big = problem.spec.input_dim * 4 >= self.BIG_ROW_BYTES
        self.feed = DmaFeed(problem, self.engine) if big else ZeroCopyFeed(problem, self.engine)
        self.h2d_bytes, self.d2h_bytes = self.feed.h2d_bytes, self.feed.d2h_bytes
        self.path = ("host SplitMix64 sampling -> per-row DMA from the pinned dataset (copy stream, overlapped) -> "
                     "(graph: round, loss D2H) -> sync" if big else
                     "(graph: device SplitMix64 sampling reading the rows from the pinned host dataset over PCIe, "
                     "round, loss D2H) -> sync")

    def step(self) -> float:
        return self.feed.step()

    def close(self) -> None:
        """Release the feed's graphs and the engine's communicator."""
        for name in ("graphs", "graph"):
            if hasattr(self.feed, name):
                setattr(self.feed, name, None if name == "graph" else [None, None])
        self.engine.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
