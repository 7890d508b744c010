"""Update rules of arXiv 1708.02983 Eq. (1)-(6) on device buffers.

``HyperParams`` is the reference's (updates.py:20-38). The functions below
keep the reference names and pure semantics (return new buffers, inputs
untouched: updates.py:3-9) on float32 CUDA tensors and run the libesgd
kernels; ``*_`` variants update in place (what the trainers use). The
kernels evaluate the reference's fp32 operation order with no FMA
contraction, so results equal the float32 reference bitwise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import check_f32, ptr, same_shape, stream_ptr
from .errors import InputError, ShapeError


@dataclass(frozen=True)
class HyperParams:
    """eta: learning rate; rho: elastic rate; mu: momentum rate.

    As in the reference, nothing normalises by worker count, so the
    synchronous full-sum center step is stable only when eta*rho*P < 1.
    """

    eta: float = 0.01
    rho: float = 0.1
    mu: float = 0.9

    def __post_init__(self):
        if self.eta <= 0:
            raise InputError(f"eta must be > 0, got {self.eta}")
        if self.rho < 0:
            raise InputError(f"rho must be >= 0, got {self.rho}")
        if not 0 <= self.mu < 1:
            raise InputError(f"mu must be in [0, 1), got {self.mu}")

    # the scalars as the fp32 reference sees them: Python floats are weak
    # scalars cast to float32 at use; eta*rho is formed in double first
    @property
    def eta32(self) -> float:
        return float(np.float32(self.eta))

    @property
    def etarho32(self) -> float:
        return float(np.float32(self.eta * self.rho))

    @property
    def mu32(self) -> float:
        return float(np.float32(self.mu))


def _n(t: torch.Tensor) -> int:
    return t.numel()


def easgd_worker_step_(w, grad, center, eta: float, rho: float) -> torch.Tensor:
    check_f32(w, grad, center)
    same_shape(w, grad, center)
    _lib.call("esgd_worker_step_f32", ptr(w), ptr(w), ptr(grad), ptr(center), _n(w),
              float(np.float32(eta)), float(np.float32(eta * rho)), stream_ptr())
    return w


def easgd_worker_step(w, grad, center, eta: float, rho: float) -> torch.Tensor:
    """W' = (W - eta*grad) - (eta*rho)*(W - center)  (updates.py:85-93)."""
    check_f32(w, grad, center)
    same_shape(w, grad, center)
    out = torch.empty_like(w)
    _lib.call("esgd_worker_step_f32", ptr(out), ptr(w), ptr(grad), ptr(center), _n(w),
              float(np.float32(eta)), float(np.float32(eta * rho)), stream_ptr())
    return out


def easgd_center_step_from_sum(center, weight_sum, num_workers: int, eta: float,
                               rho: float) -> torch.Tensor:
    """C' = C + (eta*rho)*(S - P*C)  (updates.py:113-119)."""
    check_f32(center, weight_sum)
    same_shape(center, weight_sum)
    if num_workers < 1:
        raise InputError("num_workers must be >= 1")
    out = torch.empty_like(center)
    _lib.call("esgd_center_step_from_sum_f32", ptr(out), ptr(center), ptr(weight_sum),
              _n(center), float(np.float32(eta * rho)), int(num_workers), stream_ptr())
    return out


def easgd_center_step(center, worker_snapshots, eta: float, rho: float) -> torch.Tensor:
    """Snapshot form (updates.py:96-110): C' = C + (eta*rho) * sum_i (W_i - C),
    summed in worker order on the device — bitwise the reference's fp32
    arithmetic (esgd_center_step_snapshots_f32)."""
    snaps = list(worker_snapshots)
    if not snaps:
        raise InputError("easgd_center_step needs at least one worker snapshot")
    check_f32(center, *snaps)
    for s in snaps:
        same_shape(center, s)
    S = torch.stack([s.reshape(-1) for s in snaps]).contiguous()
    out = torch.empty_like(center)
    hy = HyperParams(eta, rho)
    _lib.call("esgd_center_step_snapshots_f32", ptr(out), ptr(center), ptr(S), S.stride(0), len(snaps),
              center.numel(), hy.etarho32, stream_ptr())
    return out


def easgd_center_incremental(center, worker, eta: float, rho: float) -> torch.Tensor:
    """C' = C + (eta*rho)*(W_j - C)  (updates.py:122-131)."""
    check_f32(center, worker)
    same_shape(center, worker)
    out = torch.empty_like(center)
    _lib.call("esgd_center_incr_f32", ptr(out), ptr(center), ptr(worker), _n(center),
              float(np.float32(eta * rho)), stream_ptr())
    return out


def measgd_worker_step(w, v, grad, center, eta: float, mu: float, rho: float):
    """V' = mu*V - eta*grad; W' = (W + V') - (eta*rho)*(W - C)  (updates.py:134-140)."""
    check_f32(w, v, grad, center)
    same_shape(w, v, grad, center)
    w2, v2 = w.clone(), v.clone()
    _lib.call("esgd_measgd_update_f32", ptr(w2), ptr(v2), ptr(grad), ptr(center), _n(w),
              float(np.float32(eta)), float(np.float32(mu)), float(np.float32(eta * rho)),
              stream_ptr())
    return w2, v2


def sgd_step(w, grad, eta: float) -> torch.Tensor:
    """W' = W - eta*grad  (updates.py:71-74)."""
    check_f32(w, grad)
    same_shape(w, grad)
    out = w.clone()
    _lib.call("esgd_sgd_step_f32", ptr(out), ptr(grad), _n(w), float(np.float32(eta)), stream_ptr())
    return out


def msgd_step(w, v, grad, eta: float, mu: float):
    """V' = mu*V - eta*grad; W' = W + V'  (updates.py:77-82)."""
    check_f32(w, v, grad)
    same_shape(w, v, grad)
    w2, v2 = w.clone(), v.clone()
    _lib.call("esgd_msgd_step_f32", ptr(w2), ptr(v2), ptr(grad), _n(w), float(np.float32(eta)),
              float(np.float32(mu)), stream_ptr())
    return w2, v2


def sync_update_sum_(W: torch.Tensor, G: torch.Tensor, C: torch.Tensor, S: torch.Tensor, S_next: torch.Tensor,
                     n: int, num_workers: int, hyper: HyperParams, stream=None) -> None:
    """sync_update_ plus the next round's local replica sum S_next =
    tree_sum(W_r(t+1)) (fabric/collectives.py:18-32 order) in the same pass;
    S_next may be S."""
    if W.dim() != 2 or G.shape != W.shape:
        raise ShapeError("sync_update_sum_: W and G must be (nrep, ld) with equal shapes")
    _lib.call("esgd_sync_update_sum_f32", ptr(W), W.stride(0), ptr(G), G.stride(0), W.shape[0],
              ptr(C), ptr(S), ptr(S_next), n, hyper.eta32, hyper.etarho32, int(num_workers),
              stream_ptr(stream))


def sync_update_(W: torch.Tensor, G: torch.Tensor, C: torch.Tensor, S: torch.Tensor, n: int,
                 num_workers: int, hyper: HyperParams, stream=None) -> None:
    """Fused Sync-EASGD round update for all local replicas (rows of W/G),
    in place (trainers/synchronous.py:57-64)."""
    if W.dim() != 2 or G.shape != W.shape:
        raise ShapeError("sync_update_: W and G must be (nrep, ld) with equal shapes")
    _lib.call("esgd_sync_update_f32", ptr(W), W.stride(0), ptr(G), G.stride(0), W.shape[0],
              ptr(C), ptr(S), n, hyper.eta32, hyper.etarho32, int(num_workers),
              stream_ptr(stream))


def sync_update_solo_(W: torch.Tensor, G: torch.Tensor, C: torch.Tensor, n: int, hyper: HyperParams,
                      stream=None) -> None:
    """Round update of a one-worker run (P = 1): S = W(t), so the fused
    update reads W, G, C and writes W, C only (esgd_sync_update_solo_f32)."""
    if W.dim() != 2 or W.shape[0] != 1 or G.shape != W.shape:
        raise ShapeError("sync_update_solo_: W and G must be (1, ld)")
    _lib.call("esgd_sync_update_solo_f32", ptr(W), ptr(G), ptr(C), n, hyper.eta32, hyper.etarho32,
              stream_ptr(stream))
