"""CUDA-event timing of the conv data-movement kernels on the AlexNet b=128
layer shapes (CNHW planes), with achieved algorithmic GB/s:

    python tools/bench_conv.py

im2col: writes K*pixels floats (reads of the input hit L1/L2);
col2im: reads K*pixels floats; maxpool bwd: reads dy + argmax, writes dx.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200 import _lib  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402

B = 128
# name, C_in, H, k, stride, pad
CONVS = [("conv1", 3, 224, 11, 4, 2), ("conv2", 64, 27, 5, 1, 2), ("conv3", 192, 13, 3, 1, 1),
         ("conv4", 384, 13, 3, 1, 1), ("conv5", 256, 13, 3, 1, 1)]
POOLS = [("pool1", 64, 55), ("pool2", 192, 27), ("pool5", 256, 13)]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    lib = _lib.load()
    tot = 0.0
    for name, c, h, k, s, p in CONVS:
        oh = (h + 2 * p - k) // s + 1
        npix = B * oh * oh
        np4 = (npix + 3) // 4 * 4
        kd = c * k * k
        x = torch.randn(c * B * h * h, device="cuda")
        col = torch.empty(kd * np4, device="cuda")
        xd = _lib.cnhw(B, c, h, h, B * h * h)

        def fwd():
            _lib.check(lib.esgd_im2col_f32(col.data_ptr(), 1, np4, 0, x.data_ptr(), xd, 0, k, k, s, p, oh, oh, 1,
                                           stream_ptr()))

        def bwd():
            _lib.check(lib.esgd_col2im_f32(x.data_ptr(), xd, 0, col.data_ptr(), 1, np4, 0, k, k, s, p, oh, oh,
                                           None, 0, 1, stream_ptr()))

        t = timeit(fwd)
        tot += t
        print(f"im2col {name:6s} K={kd:5d} pix={npix:7d} {t:8.1f} us {kd * npix * 4 / t / 1e3:7.0f} GB/s")
        if name != "conv1":
            t = timeit(bwd)
            tot += t
            print(f"col2im {name:6s} K={kd:5d} pix={npix:7d} {t:8.1f} us {kd * npix * 4 / t / 1e3:7.0f} GB/s")
        del x, col
    for name, c, h in POOLS:
        oh = (h - 3) // 2 + 1
        x = torch.randn(c * B * h * h, device="cuda")
        y = torch.empty(c * B * oh * oh, device="cuda")
        am = torch.empty(c * B * oh * oh, dtype=torch.int32, device="cuda")
        xd, yd = _lib.cnhw(B, c, h, h, B * h * h), _lib.cnhw(B, c, oh, oh, B * oh * oh)

        def pf():
            _lib.check(lib.esgd_maxpool_fwd_f32(y.data_ptr(), yd, 0, am.data_ptr(), x.data_ptr(), xd, 0, 3, 2, 0, 1,
                                                stream_ptr()))

        def pb():
            _lib.check(lib.esgd_maxpool_bwd_f32(x.data_ptr(), xd, 0, y.data_ptr(), yd, 0, am.data_ptr(), None, 0,
                                                3, 2, 0, 1, stream_ptr()))

        t = timeit(pf)
        tot += t
        by = (x.numel() + 2 * y.numel()) * 4
        print(f"poolF  {name:6s} in={x.numel():9d} {t:8.1f} us {by / t / 1e3:7.0f} GB/s")
        t = timeit(pb)
        tot += t
        by = (x.numel() + 2 * y.numel()) * 4
        print(f"poolB  {name:6s} in={x.numel():9d} {t:8.1f} us {by / t / 1e3:7.0f} GB/s")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    torch.cuda.set_device(0)
    main()
