"""Device plumbing: torch CUDA tensors as HBM buffers, the current stream as
a raw cudaStream_t for libesgd, and the fp32 contract checks."""

from __future__ import annotations

import torch

from . import _lib
from .errors import CudaError, ShapeError

F32 = torch.float32


def require_cuda(device=None) -> torch.device:
    """The device engine has no CPU fallback: fail loudly without a B200."""
    if not torch.cuda.is_available():
        raise CudaError("engine 'cuda' needs a CUDA device (B200, sm_100a); none is visible")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       torch.device(device).index or 0)
    lib = _lib.load()
    if not lib.esgd_device_ok(dev.index):
        raise CudaError(_lib.last_error())
    return dev


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def check_f32(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda or t.dtype != F32:
            raise ShapeError(f"expected a float32 CUDA tensor, got {t.dtype} on {t.device}")
        if not t.is_contiguous():
            raise ShapeError("expected a contiguous tensor")


def same_shape(*ts: torch.Tensor) -> None:
    shapes = {tuple(t.shape) for t in ts}
    if len(shapes) > 1:
        raise ShapeError(f"buffer shape mismatch: {sorted(shapes)}")


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m
