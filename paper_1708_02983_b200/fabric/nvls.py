"""Symmetric-memory plumbing for the fused multi-GPU round update over NVLink
SHARP multicast (csrc/nvls.cu).

PyTorch's symmetric memory (``torch.distributed._symmetric_memory``) maps
one allocation per rank and a multicast address that spans all of them
(NVSwitch multicast objects); the round's collective + update is then ONE
libesgd kernel (``esgd_sync_update_nvls_f32``) preceded by a device-side
cross-GPU barrier (``esgd_nvls_barrier``) — no NCCL call in the round.

Layout (one symmetric fp32 allocation of 4*ld per rank): S[0], S[1] (this
rank's replica sums, double-buffered by round parity) and C[0], C[1] (the
center, written by every rank's multicast broadcast of its slice).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .. import _lib
from ..device import stream_ptr
from ..errors import CudaError


def nvls_wanted() -> bool:
    return os.environ.get("ESGD_NVLS", "1") != "0"


def nvls_reserve_sms() -> int:
    """SMs the overlapped center kernel takes for itself while the GEMMs use
    the rest (ESGD_NVLS_RESERVE; default 0 = small center CTAs on every SM,
    co-resident with the GEMM CTAs). Measured at N = 2 (AlexNet, B200): 8
    reserved SMs make the round 10% slower (4.84 -> 5.34 ms): the GEMMs on 140
    SMs lose more than the 5% of SMs (whole extra waves of tiles) and the
    center on 8 SMs takes 1.4 ms instead of 0.7 (tools/nvls_timeline.py)."""
    return int(os.environ.get("ESGD_NVLS_RESERVE", "0"))


def nvls_center_ctas() -> int:
    r = nvls_reserve_sms()
    return -r if r > 0 else int(os.environ.get("ESGD_NVLS_CTAS", "148"))


def nvls_fused_single_kernel() -> bool:
    """ESGD_NVLS=fused: center + workers in one kernel after the backward
    (measured slower than the default split, which overlaps the center's
    NVLink traffic with the forward/backward)."""
    return os.environ.get("ESGD_NVLS", "1") == "fused"


class NvlsRound:
    """Symmetric S/C buffers, their multicast addresses and the barrier flags
    of one rank; ``update(...)`` enqueues barrier + fused update for a round."""

    def __init__(self, ld: int, device, group=None):
        import torch.distributed._symmetric_memory as symm

        if ld % 4:
            raise CudaError("nvls: padded length must be a multiple of 4")
        group = group or dist.group.WORLD
        gname = group.group_name
        self.ld = ld
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.buf = symm.empty(4 * ld, dtype=torch.float32, device=device)
        self.buf.zero_()
        self.h = symm.rendezvous(self.buf, gname)
        if not self.h.multicast_ptr:
            raise CudaError("nvls: no multicast support on this device/fabric")
        self.flags = symm.empty(64, dtype=torch.int32, device=device)
        self.flags.zero_()
        self.hf = symm.rendezvous(self.flags, gname)
        torch.cuda.synchronize()
        dist.barrier(group=group)
        # multicast address of this tensor = multicast base + its offset in the allocation
        off = self.buf.data_ptr() - self.h.buffer_ptrs[self.rank]
        self.mc = self.h.multicast_ptr + off
        foff = self.flags.data_ptr() - self.hf.buffer_ptrs[self.rank]
        self.peer_flags = torch.tensor([p + foff for p in self.hf.buffer_ptrs], dtype=torch.int64, device=device)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        self.S = [self.buf[0:ld], self.buf[ld:2 * ld]]
        self.C = [self.buf[2 * ld:3 * ld], self.buf[3 * ld:4 * ld]]
        self.S_mc = [self.mc, self.mc + 4 * ld]
        self.C_mc = [self.mc + 8 * ld, self.mc + 12 * ld]

    def barrier(self, stream=None) -> None:
        _lib.call("esgd_nvls_barrier", self.peer_flags.data_ptr(), self.world, self.rank, self.epoch.data_ptr(),
                  stream_ptr(stream))

    def center(self, parity: int, num_workers: int, hyper, stream=None, ctas: int | None = None) -> None:
        """Side-stream half of round parity p: barrier, then this rank's slice
        of C[p^1] = center step of C[p] with the all-rank sum of S[p]
        (NVSwitch ld_reduce), broadcast to every rank (multicast store)."""
        p = parity & 1
        if ctas is None:
            ctas = nvls_center_ctas()
        self.barrier(stream)
        _lib.call("esgd_center_step_nvls_f32", self.C[p].data_ptr(), self.S_mc[p], self.C_mc[p ^ 1], self.ld,
                  self.world, self.rank, hyper.etarho32, int(num_workers), ctas, stream_ptr(stream))

    def workers(self, W: torch.Tensor, G: torch.Tensor, parity: int, hyper, stream=None) -> None:
        """Local half: worker step against C[p], S[p^1] = replica sum of the new W."""
        p = parity & 1
        _lib.call("esgd_worker_step_sum_f32", W.data_ptr(), W.stride(0), G.data_ptr(), G.stride(0), W.shape[0],
                  self.C[p].data_ptr(), self.S[p ^ 1].data_ptr(), self.ld, hyper.eta32, hyper.etarho32,
                  stream_ptr(stream))

    def update(self, W: torch.Tensor, G: torch.Tensor, parity: int, num_workers: int, hyper, stream=None) -> None:
        """Round with parity p: barrier, then C[p^1] = center step of C[p] with
        the all-rank sum of S[p] (this rank's slice, broadcast), W = worker step
        against C[p], S[p^1] = local replica sum of the new W."""
        p = parity & 1
        self.barrier(stream)
        _lib.call("esgd_sync_update_nvls_f32", W.data_ptr(), W.stride(0), G.data_ptr(), G.stride(0), W.shape[0],
                  self.C[p].data_ptr(), self.S_mc[p], self.C_mc[p ^ 1], self.S[p ^ 1].data_ptr(), self.ld,
                  self.world, self.rank, hyper.eta32, hyper.etarho32, int(num_workers), stream_ptr(stream))
