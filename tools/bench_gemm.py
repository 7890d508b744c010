"""tcgen05 GEMM throughput on the AlexNet contractions (CUDA events, warm).

    python tools/bench_gemm.py [--precision 3] [--only NAME]
Reports fp32-equivalent TFLOP/s (2*M*N*K / t) and the tf32 tensor-pipe rate
(x3 for 3xTF32)."""

import argparse
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200 import _lib  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402

# (name, m, n, k, a_major, b_major, c_mcontig) of AlexNet b=128 as the CNHW
# engine issues them (nets.py): conv outputs / dcolT are M-contiguous
SHAPES = [
    ("conv1.fwd", 387200, 64, 363, 1, 0, 1),
    ("conv2.fwd", 93312, 192, 1600, 1, 0, 1),
    ("conv3.fwd", 21632, 384, 1728, 1, 0, 1),
    ("conv2.wgrad", 192, 1600, 93312, 0, 0, 0),
    ("conv1.wgrad", 64, 363, 387200, 0, 0, 0),
    ("conv2.dgrad", 93312, 1600, 192, 1, 0, 1),
    ("conv4.dgrad", 21632, 3456, 256, 1, 0, 1),
    ("fc6.fwd", 128, 4096, 9216, 0, 1, 0),
    ("fc6.wgrad", 9216, 4096, 128, 1, 0, 0),
    ("fc6.dgrad", 128, 9216, 4096, 0, 0, 0),
    ("fc7.wgrad", 4096, 4096, 128, 1, 0, 0),
    # exploration: the short-K problems with the big operand as B instead
    ("x.conv2.dgradT", 1600, 93312, 192, 0, 1, 0),
    ("x.fc6.wgradT", 4096, 9216, 128, 0, 1, 1),
    ("x.conv2.dgrad.kmajor", 93312, 1600, 192, 0, 0, 1),
    ("x.conv2.dgrad.rowmajorC", 93312, 1600, 192, 1, 0, 0),
    # forward convolutions as C^T = W . colT (the weights as the K-major A operand)
    ("conv4.fwd", 21632, 256, 3456, 1, 0, 1),
    ("x.conv4.fwdT", 256, 21632, 3456, 0, 1, 0),
    ("conv5.fwd", 21632, 256, 2304, 1, 0, 1),
    ("x.conv5.fwdT", 256, 21632, 2304, 0, 1, 0),
    ("x.conv3.fwdT", 384, 21632, 1728, 0, 1, 0),
    ("x.conv2.fwdT", 192, 93312, 1600, 0, 1, 0),
    # conv1 with a K-major (pixel-row) im2col matrix: forward A K-major, wgrad B MN-major
    ("x.conv1.fwd.kmajor", 387200, 64, 363, 0, 0, 1),
    ("x.conv1.wgrad.bmn", 64, 363, 387200, 0, 1, 0),
    ("x.conv2.fwd.kmajor", 93312, 192, 1600, 0, 0, 1),
    ("x.conv2.wgrad.bmn", 192, 1600, 93312, 0, 1, 0),
]


def run(name, m, n, k, am, bm, cm, precision, reps=10):
    kp = (k + 3) // 4 * 4
    mp = (m + 3) // 4 * 4
    np_ = (n + 3) // 4 * 4
    A = torch.randn((kp * mp,), device="cuda")
    B = torch.randn((kp * np_,), device="cuda")
    Cm = torch.empty((m * n,), device="cuda")
    ws = torch.zeros(1 << 24, device="cuda")  # (split-K tile counters start at zero)
    lda = mp if am else kp
    ldb = np_ if bm else kp
    c_sm, c_sn = (1, mp) if cm else (np_, 1)
    Cm = torch.empty((mp * np_,), device="cuda")
    d = _lib.TcGemmDesc(m, n, k, 1, A.data_ptr(), lda, 0, B.data_ptr(), ldb, 0, Cm.data_ptr(), c_sm, c_sn, 0,
                        None, 0, None, 0, 0, 0, 0, 0, precision, am, bm, ws.data_ptr(), ws.numel())
    lib = _lib.load()
    for _ in range(3):
        _lib.check(lib.esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _lib.check(lib.esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    fl = 2.0 * m * n * k
    print(f"{name:12s} m={m:7d} n={n:5d} k={k:7d} maj=({am},{bm})  {t * 1e3:8.3f} ms  "
          f"{fl / t / 1e12:7.1f} TFLOP/s fp32-eq  {precision * fl / t / 1e12:7.1f} TFLOP/s tf32-pipe")
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", type=int, default=3)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    tot = 0.0
    for s in SHAPES:
        if args.only and args.only not in s[0]:
            continue
        tot += run(*s, args.precision)
    print(f"total {tot * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
