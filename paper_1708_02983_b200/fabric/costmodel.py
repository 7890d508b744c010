"""alpha-beta cost model (reference fabric/costmodel.py:27-132), kept so that
``run_trainer(cfg, problem, cost_model)`` accepts the same arguments, plus
its recalibration on B200: ``calibrate_allreduce`` fits
alpha and beta to measured allreduce times of the packed buffer over
NVLink/NVSwitch, ``device_compute`` measures the round's forward/backward
with CUDA events, and ``predict_sync_round`` extrapolates the Sync-EASGD
round (compute overlapped with the center collective, sync-easgd3) to GPU
counts that cannot be measured here. The device engine itself measures real
time and does not consult the model.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable

from ..errors import InputError

ComputeFn = Callable[[int, int, int], float]


def constant_compute(seconds: float) -> ComputeFn:
    def model(worker: int, batch_size: int, n_weights: int) -> float:
        return seconds
    return model


def measured_compute(run_minibatch: Callable[[], None], repeats: int = 3) -> ComputeFn:
    """reference costmodel.py:39-50: median host wall time of run_minibatch."""
    run_minibatch()
    samples = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        run_minibatch()
        samples.append(time.perf_counter() - t0)
    samples.sort()
    return constant_compute(samples[len(samples) // 2])


@dataclass(frozen=True)
class CostModel:
    alpha: float
    beta: float
    compute: ComputeFn = field(default_factory=lambda: constant_compute(0.0))
    worker_update: Callable[[int], float] = lambda n_weights: 0.0
    master_update: Callable[[int], float] = lambda n_weights: 0.0
    group_speedup: Callable[[int], float] = lambda groups: 1.0

    def __post_init__(self):
        if self.alpha < 0 or self.beta < 0:
            raise InputError("alpha and beta must be >= 0")

    @classmethod
    def preset(cls, name: str, **overrides) -> "CostModel":
        try:
            alpha, beta = _PRESETS[name]
        except KeyError:
            raise InputError(f"unknown cost preset {name!r}; have {sorted(_PRESETS)}")
        return cls(alpha=alpha, beta=beta, **overrides)

    def message_seconds(self, nbytes: int) -> float:
        return message_cost(nbytes, self)


# measured on this pool's HGX B200 (NVLink 5 / NVSwitch): ncclAllReduce of the
# packed fp32 buffer, fitted by calibrate_allreduce (profiles/r01_costmodel.md)
B200_NVLINK_ALPHA = 29.1e-6
B200_NVLINK_BETA = 1.0 / 407.7e9

_PRESETS = {
    "fdr": (0.7e-6, 0.2e-9),
    "qdr": (1.2e-6, 0.3e-9),
    "10gbe": (7.2e-6, 0.9e-9),
    "b200-nvlink": (B200_NVLINK_ALPHA, B200_NVLINK_BETA),
}
PRESET_NAMES = tuple(sorted(_PRESETS))


def message_cost(nbytes: int, cm: CostModel) -> float:
    if nbytes < 0:
        raise InputError(f"message size must be >= 0, got {nbytes}")
    return cm.alpha + cm.beta * nbytes


def tree_depth(participants: int) -> int:
    if participants < 1:
        raise InputError("participants must be >= 1")
    return math.ceil(math.log2(participants)) if participants > 1 else 0


@dataclass(frozen=True)
class PackedComparison:
    """reference costmodel.py:107-121: one packed message vs one per layer;
    per_layer = packed + (L - 1) * alpha by construction."""

    packed: float
    per_layer: float
    latency_overhead: float


def packed_vs_perlayer_cost(layer_sizes, cm: CostModel) -> PackedComparison:
    sizes = list(layer_sizes)
    if not sizes:
        raise InputError("need at least one layer")
    total = sum(sizes)
    packed = cm.alpha + cm.beta * total
    overhead = (len(sizes) - 1) * cm.alpha
    return PackedComparison(packed, packed + overhead, overhead)


# ---- B200 recalibration ---------------------------------------

def fit_alpha_beta(sizes_bytes, seconds) -> tuple[float, float]:
    """Least-squares fit of t = alpha + beta * bytes (alpha, beta >= 0)."""
    n = len(sizes_bytes)
    if n < 2 or n != len(seconds):
        raise InputError("need >= 2 (size, time) samples")
    mx = sum(sizes_bytes) / n
    my = sum(seconds) / n
    sxx = sum((x - mx) ** 2 for x in sizes_bytes)
    sxy = sum((x - mx) * (y - my) for x, y in zip(sizes_bytes, seconds))
    beta = max(0.0, sxy / sxx) if sxx > 0 else 0.0
    alpha = max(0.0, my - beta * mx)
    return alpha, beta


def calibrate_allreduce(sizes_bytes=(4 << 10, 1 << 20, 16 << 20, 64 << 20, 256 << 20), reps: int = 10,
                        group=None) -> tuple[CostModel, list[tuple[int, float]]]:
    """Time ncclAllReduce(sum, fp32) of each payload size on the current
    process group with CUDA events (max over ranks), fit alpha/beta.
    Collective: every rank must call it."""
    import torch
    import torch.distributed as dist

    samples = []
    for nb in sizes_bytes:
        x = torch.ones(max(1, nb // 4), dtype=torch.float32, device="cuda")
        for _ in range(3):
            dist.all_reduce(x, group=group)
        torch.cuda.synchronize()
        dist.barrier(group=group)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            dist.all_reduce(x, group=group)
        b.record()
        b.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 1e3 / reps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        samples.append((nb, float(t.item())))
    alpha, beta = fit_alpha_beta([s for s, _ in samples], [t for _, t in samples])
    return CostModel(alpha=alpha, beta=beta), samples


def device_compute(engine, rounds: int = 5) -> ComputeFn:
    """Calibrate the compute model from the device: CUDA-event time of the
    engine's gradient pass (forward + backward of all local replicas)."""
    import torch

    from ..device import stream_ptr

    G, W = engine.G.clone(), engine.W.clone()
    engine.plan.gradient(G, W, stream_ptr())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(rounds):
        engine.plan.gradient(G, W, stream_ptr())
    b.record()
    b.synchronize()
    return constant_compute(a.elapsed_time(b) / 1e3 / rounds)


def predict_sync_round(cm: CostModel, compute_seconds: float, n_params: int, gpus: int,
                       update_seconds: float = 0.0, interference: float = 0.0) -> dict:
    """Sync-EASGD3 round on ``gpus`` GPUs (one worker each): the center
    collective (a ring allreduce of the packed fp32 buffer: 2(N-1)/N of the
    payload per rank, plus alpha per step) overlaps the forward/backward;
    ``interference`` is the fraction of the collective's time the overlap
    costs the compute (measured: ~0.3-0.5 of it on B200). Returns seconds,
    samples-per-second multiplier and weak-scaling efficiency vs 1 GPU."""
    if gpus < 1:
        raise InputError("gpus must be >= 1")
    payload = 4 * n_params
    comm = 0.0 if gpus == 1 else (2 * (gpus - 1) * cm.alpha + 2 * (gpus - 1) / gpus * payload * cm.beta)
    exposed = max(0.0, comm - compute_seconds)
    round_s = compute_seconds + interference * min(comm, compute_seconds) + exposed + update_seconds
    base = compute_seconds + update_seconds
    return {"round_seconds": round_s, "comm_seconds": comm, "exposed_comm_seconds": exposed,
            "weak_scaling_efficiency": base / round_s}
