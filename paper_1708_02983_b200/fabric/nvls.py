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
    return os.environ.get("ESGD_NVLS", "ce") != "0"


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


def nvls_copy_engines() -> bool:
    """Default (ESGD_NVLS unset or "ce"): the center slice's NVLink traffic on
    the copy engines (cudaMemcpyAsync of peer slices + a local sum / center
    kernel). ESGD_NVLS=1: multimem ld_reduce / st from SM threads, which
    co-run with the forward / backward's GEMM CTAs and slow them (measured at
    N = 2, AlexNet: round 4.83 ms, exposed 10.3%, vs 4.55 ms, 3.1% here)."""
    return os.environ.get("ESGD_NVLS", "ce") == "ce"


def nvls_fused_single_kernel() -> bool:
    """ESGD_NVLS=fused: center + workers in one kernel after the backward
    (measured slower than the default split, which overlaps the center's
    NVLink traffic with the forward/backward)."""
    return os.environ.get("ESGD_NVLS", "ce") == "fused"


class NvlsRound:
    """Symmetric S/C buffers, their multicast addresses and the barrier flags
    of one rank; ``update(...)`` enqueues barrier + fused update for a round."""

    def __init__(self, ld: int, device, group=None, nrep: int = 0):
        import torch.distributed._symmetric_memory as symm

        if ld % 4:
            raise CudaError("nvls: padded length must be a multiple of 4")
        group = group or dist.group.WORLD
        gname = group.group_name
        self.ld = ld
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        # copy-engine path with one worker per rank: the worker buffer W itself
        # lives in the symmetric allocation too (after S[0], S[1], C[0], C[1]),
        # its peers read their slice of it directly — no local sum S to form
        self.w_src = nvls_copy_engines() and nrep == 1
        self.buf = symm.empty((5 if self.w_src else 4) * ld, dtype=torch.float32, device=device)
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
        self.W = self.buf[4 * ld:5 * ld].view(1, ld) if self.w_src else None
        # copy-engine variant: this rank's slice [lo, hi) (floats, multiple of
        # 4) of every rank's S lands in recv[j]; peers' buffers by address
        self.ce = nvls_copy_engines()
        per = (ld // 4 + self.world - 1) // self.world
        self.lo, self.hi = min(ld, 4 * per * self.rank), min(ld, 4 * per * (self.rank + 1))
        if self.ce:
            if self.world > 8:
                raise CudaError("nvls ce: at most 8 ranks")
            self.peer = [p + off for p in self.h.buffer_ptrs]  # each rank's copy of self.buf
            self.recv = torch.empty((self.world, max(4, self.hi - self.lo)), dtype=torch.float32, device=device)
            srcs = []
            for q in range(2):
                own = (self.W if self.w_src else self.S[q]).data_ptr() + 4 * self.lo
                srcs.append([own if j == self.rank else self.recv[j].data_ptr() for j in range(self.world)])
            self.srcs = torch.tensor(srcs, dtype=torch.int64, device=device)

    def barrier(self, stream=None) -> None:
        _lib.call("esgd_nvls_barrier", self.peer_flags.data_ptr(), self.world, self.rank, self.epoch.data_ptr(),
                  stream_ptr(stream))

    def center(self, parity: int, num_workers: int, hyper, stream=None, ctas: int | None = None) -> None:
        """Side-stream half of round parity p: barrier, then this rank's slice
        of C[p^1] = center step of C[p] with the all-rank sum of S[p]
        (NVSwitch ld_reduce), broadcast to every rank (multicast store)."""
        p = parity & 1
        if self.ce:
            self.center_ce(p, num_workers, hyper, stream)
            return
        if ctas is None:
            ctas = nvls_center_ctas()
        self.barrier(stream)
        _lib.call("esgd_center_step_nvls_f32", self.C[p].data_ptr(), self.S_mc[p], self.C_mc[p ^ 1], self.ld,
                  self.world, self.rank, hyper.etarho32, int(num_workers), ctas, stream_ptr(stream))

    def center_ce(self, p: int, num_workers: int, hyper, stream=None) -> None:
        """Copy-engine center slice of round parity p: barrier; pull this
        rank's slice of every peer's S[p] (or, one worker per rank, of its W:
        then a second barrier, after which the ranks' worker steps may
        overwrite W) with cudaMemcpyAsync over NVLink; sum in rank order +
        center step into C[p^1]'s slice; push it to every peer."""
        self.barrier(stream)
        n = self.hi - self.lo
        sp = stream_ptr(stream)
        s_off = 4 * ((4 if self.w_src else p) * self.ld + self.lo)
        c_off = 4 * ((2 + (p ^ 1)) * self.ld + self.lo)
        for j in range(self.world):
            if j != self.rank and n > 0:
                _lib.call("esgd_copy_async", self.recv[j].data_ptr(), self.peer[j] + s_off, 4 * n, sp)
        if self.w_src:
            self.barrier(stream)
        if n <= 0:
            return
        _lib.call("esgd_center_step_sum_f32", self.C[p].data_ptr() + 4 * self.lo, self.srcs[p].data_ptr(),
                  self.world, self.C[p ^ 1].data_ptr() + 4 * self.lo, n, hyper.etarho32, int(num_workers), sp)
        for j in range(self.world):
            if j != self.rank:
                _lib.call("esgd_copy_async", self.peer[j] + c_off, self.C[p ^ 1].data_ptr() + 4 * self.lo, 4 * n, sp)

    def workers(self, W: torch.Tensor, G: torch.Tensor, parity: int, hyper, stream=None) -> None:
        """Local half: worker step against C[p], S[p^1] = replica sum of the new
        W (one worker per rank on the copy-engine path: the worker step alone,
        16 B/param, in place on the symmetric W)."""
        p = parity & 1
        if self.w_src:
            _lib.call("esgd_worker_step_f32", W.data_ptr(), W.data_ptr(), G.data_ptr(), self.C[p].data_ptr(),
                      self.ld, hyper.eta32, hyper.etarho32, stream_ptr(stream))
            return
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
