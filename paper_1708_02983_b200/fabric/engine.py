"""Breakdown categories (reference fabric/engine.py:33-41) and the lock-free
center apply (fabric/engine.py:156-166) on the device."""

from __future__ import annotations

import torch

from .. import _lib
from ..device import check_f32, ptr, same_shape, stream_ptr
from ..errors import ShapeError

CATEGORIES = (
    "peer_param",
    "data_stage",
    "master_param",
    "forward_backward",
    "worker_update",
    "master_update",
)
COMM_CATEGORIES = ("peer_param", "data_stage", "master_param")


def hogwild_apply(center: torch.Tensor, delta: torch.Tensor) -> None:
    """``center += delta`` with no buffer lock: vector red.global.add per
    4 floats, concurrent callers on other streams interleave per element."""
    check_f32(center, delta)
    if center.shape != delta.shape:
        raise ShapeError(f"hogwild_apply shape mismatch: {tuple(center.shape)} vs {tuple(delta.shape)}")
    _lib.call("esgd_hogwild_axpy_f32", ptr(center), ptr(delta), center.numel(), 1.0, stream_ptr())


def hogwild_elastic_apply(center: torch.Tensor, w: torch.Tensor, snap: torch.Tensor,
                          etarho32: float, stream=None) -> None:
    """center += (eta*rho)*(w - snap), lock-free (trainers/hogwild.py:180)."""
    _lib.call("esgd_hogwild_apply_f32", ptr(center), ptr(w), ptr(snap), w.numel(), etarho32,
              stream_ptr(stream))
