"""The center sum: fixed-order replica reduction on the device plus the NCCL
allreduce across processes (replaces fabric/collectives.py:18-32 tree_sum,
trainers/synchronous.py:59)."""

from __future__ import annotations

import torch
import torch.distributed as dist

from .. import _lib
from ..device import check_f32, ptr, stream_ptr
from ..errors import InputError, ShapeError


def tree_sum(buffers) -> torch.Tensor:
    """Elementwise sum of equal-shape device buffers in the reference's
    binomial order (partial[pos] += partial[pos+distance], distance doubling);
    inputs are not modified."""
    bufs = list(buffers)
    if not bufs:
        raise InputError("tree_sum needs at least one buffer")
    shapes = {tuple(b.shape) for b in bufs}
    if len(shapes) > 1:
        raise ShapeError(f"buffer shape mismatch: {sorted(shapes)}")
    check_f32(*bufs)
    n = bufs[0].numel()
    stacked = torch.stack([b.reshape(-1) for b in bufs])
    out = torch.empty(n, dtype=torch.float32, device=bufs[0].device)
    if len(bufs) > 64:
        # binomial order over blocks of 64 is not the reference's order; keep exactness simple
        raise InputError("tree_sum over more than 64 device buffers is not supported")
    _lib.call("esgd_replica_tree_sum_f32", ptr(out), ptr(stacked), stacked.stride(0), len(bufs), n,
              stream_ptr())
    return out.reshape(bufs[0].shape)


def replica_sum_(S: torch.Tensor, W: torch.Tensor, n: int, stream=None) -> None:
    """S[:n] = binomial-order sum of the rows of W (local replicas)."""
    _lib.call("esgd_replica_tree_sum_f32", ptr(S), ptr(W), W.stride(0), W.shape[0], n,
              stream_ptr(stream))


def local_workers(workers: int, world_size: int, rank: int) -> range:
    """Workers owned by ``rank``: a contiguous block of workers/world_size, so
    the local fixed-order partial sums compose into the reference's binomial
    order whenever the block size is a power of two."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise InputError(f"bad rank {rank} of {world_size}")
    if workers % world_size:
        raise InputError(f"workers ({workers}) must be a multiple of the process count ({world_size})")
    per = workers // world_size
    return range(rank * per, (rank + 1) * per)


class CabiComm:
    """The packed-buffer allreduce through libesgd's own NCCL communicator
    (esgd_nccl_init / esgd_allreduce_sum_f32, include/esgd.h) — the path a
    host without torch.distributed uses; here torch.distributed only ships
    the 128-byte id from rank 0. Selected with ESGD_COLLECTIVE=cabi."""

    def __init__(self, device, group=None):
        import ctypes as C

        w, r = world()
        if w < 2:
            raise InputError("CabiComm needs an initialised process group of >= 2 ranks")
        lib = _lib.load()
        if not lib.esgd_nccl_available():
            raise InputError("libnccl.so.2 is not loadable")
        uid = (C.c_ubyte * 128)()
        if r == 0:
            _lib.check(lib.esgd_nccl_unique_id(C.cast(uid, C.c_void_p)), "nccl_unique_id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        self.comm = C.c_void_p()
        with torch.cuda.device(device):
            _lib.check(lib.esgd_nccl_init(C.byref(self.comm), C.cast(uid, C.c_void_p), w, r), "nccl_init")
        self.world, self.rank = w, r

    def allreduce_sum_(self, S: torch.Tensor, stream=None) -> None:
        check_f32(S)
        _lib.call("esgd_allreduce_sum_f32", self.comm, ptr(S), S.numel(), stream_ptr(stream))

    def close(self) -> None:
        if self.comm:
            _lib.call("esgd_nccl_destroy", self.comm)
            self.comm = None


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def allreduce_sum_(S: torch.Tensor, group=None) -> None:
    """In-place NCCL sum over all ranks (NVLink/NVSwitch; NVLS when NCCL picks
    it). Issued on the caller's current stream context by torch.distributed."""
    if world()[0] > 1:
        dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
