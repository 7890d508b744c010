"""Probe: does tcgen05.mma kind::tf32 ignore (truncate) the low 13 mantissa
bits of fp32 operands, or round them? Runs esgd_tc_gemm_f32 with precision=1
(single TF32 pass, raw fp32 operands) on raw, truncated and RN-rounded copies
of the same operands and compares the outputs bitwise.

    python tools/probe_tf32.py
"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200 import _lib  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402


def gemm(A, B, m, n, k):
    Cm = torch.zeros(m * n, device="cuda")
    ws = torch.zeros(1 << 20, device="cuda")
    # A K-major [m][k], B K-major [n][k], C N-contiguous [m][n]
    d = _lib.TcGemmDesc(m, n, k, 1, A.data_ptr(), k, 0, B.data_ptr(), k, 0, Cm.data_ptr(), n, 1, 0,
                        None, 0, None, 0, 0, 0, 0, 0, 1, 0, 0, ws.data_ptr(), ws.numel())
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    torch.cuda.synchronize()
    return Cm.view(m, n)


def trunc(x):
    return (x.view(torch.int32) & -8192).view(torch.float32)


def rna(x):
    i = x.view(torch.int32)
    return ((i + 4096) & -8192).view(torch.float32)


if __name__ == "__main__":
    torch.manual_seed(0)
    m, n, k = 128, 128, 8
    A = torch.randn(m * k, device="cuda")
    B = torch.randn(n * k, device="cuda")
    raw = gemm(A, B, m, n, k)
    tr = gemm(trunc(A), trunc(B), m, n, k)
    rn = gemm(rna(A), rna(B), m, n, k)
    print("raw == truncated operands:", torch.equal(raw, tr), "max diff", (raw - tr).abs().max().item())
    print("raw == RN-rounded operands:", torch.equal(raw, rn), "max diff", (raw - rn).abs().max().item())
