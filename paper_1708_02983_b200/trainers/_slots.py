"""Per-worker device state for the asynchronous schedules: each worker owns a
stream, a weight row, a gradient row, optional velocity / snapshot rows and
its own gradient plan (SplitMix64 stream, workspaces). Workers may live on
different devices; the center lives on the master device."""

from __future__ import annotations

import warnings

import numpy as np
import torch

from ..device import round_up, stream_ptr
from ..rng import stream_seed


class WorkerSlot:
    def __init__(self, wid: int, problem, init: np.ndarray, device: torch.device, batch_size: int,
                 seed: int, momentum: bool, snapshot: bool, use_tc: bool = True):
        self.wid, self.device = wid, device
        n = init.size
        self.n, self.ld = n, round_up(n, 64)
        with torch.cuda.device(device):
            self.W = torch.zeros((1, self.ld), dtype=torch.float32, device=device)
            self.W[0, :n] = torch.from_numpy(init).to(device)
            self.G = torch.zeros_like(self.W)
            self.V = torch.zeros_like(self.W) if momentum else None
            self.snap = torch.zeros(self.ld, dtype=torch.float32, device=device) if snapshot else None
            self.stream = torch.cuda.Stream(device=device)
            self.plan = problem.bind(device, 1, batch_size, self.ld, use_tc=use_tc)
            self.plan.set_streams([stream_seed(seed, wid)])
        self.done = 0
        self.graph = None
        self.no_graph = False
        self.calls = 0

    @property
    def s(self) -> int:
        return stream_ptr(self.stream)

    def gradient(self) -> None:
        """Enqueue this worker's sample + forward/backward on its stream. After
        one eager call the sequence is captured as a CUDA graph (the sampling
        kernel advances the worker's RNG counter on the device, so replays draw
        the next batches): a replay is one host call instead of ~30 launches,
        which is what bounds the asynchronous schedules' throughput."""
        with torch.cuda.device(self.device):
            if self.graph is None and self.calls >= 1 and not self.no_graph:
                self._capture()
            if self.graph is not None:
                with torch.cuda.stream(self.stream):
                    self.graph.replay()
            else:
                self.plan.gradient(self.G, self.W, self.s)
            self.calls += 1

    def prepare_graph(self) -> None:
        """Capture the gradient graph now (no execution). Capturing
        synchronises the device, so it must happen before a persistent kernel
        that depends on this worker's progress (the async device master) runs."""
        if self.graph is None:
            with torch.cuda.device(self.device):
                self._capture()
            self.calls = max(self.calls, 1)

    def _capture(self) -> None:
        rng = getattr(self.plan, "rng", None)
        before = rng.state.clone() if rng is not None else None
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(self.stream)
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                self.plan.gradient(self.G, self.W, stream_ptr(side))
        except Exception as exc:  # capture unsupported: stay eager
            warnings.warn(f"worker {self.wid}: CUDA graph capture failed ({exc}); running eagerly",
                          RuntimeWarning, stacklevel=2)
            torch.cuda.synchronize(self.device)
            self.no_graph = True
            return
        self.stream.wait_stream(side)
        if before is not None:  # capture does not execute; keep the RNG where it was
            rng.state.copy_(before)
        self.graph = g

    def w(self) -> torch.Tensor:
        return self.W[0, :self.n]


def split_iterations(total: int, workers: int) -> list[int]:
    """trainers/asynchronous.py:51-54"""
    base = total // workers
    return [base + (1 if w < total % workers else 0) for w in range(workers)]


def worker_devices(workers: int) -> list[torch.device]:
    """Workers spread round-robin over the visible GPUs (one process)."""
    n = torch.cuda.device_count()
    return [torch.device("cuda", w % n) for w in range(workers)]
