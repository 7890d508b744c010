"""Max-pool backward on AlexNet's pool shapes (b = 128, CNHW): the input-mask
form vs the pooled-output-gated form (CUDA events, warm, L2-cold inputs).

    ESGD_POOL_TILE=0 python tools/bench_pool.py   # register-gather kernels
    python tools/bench_pool.py                    # shared-memory tile kernel
"""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200 import _lib  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402

SHAPES = [("pool1", 64, 55), ("pool2", 192, 27), ("pool5", 256, 13)]


def main():
    n, k, s = 128, 3, 2
    flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    for name, c, h in SHAPES:
        oh = (h - k) // s + 1
        plane, oplane = (n * h * h + 3) // 4 * 4, (n * oh * oh + 3) // 4 * 4
        x = torch.relu(torch.randn((c, plane), device="cuda"))
        y = torch.empty((c, oplane), device="cuda")
        am = torch.empty((n, c, oh, oh), dtype=torch.int32, device="cuda")
        dy = torch.randn((c, oplane), device="cuda")
        dx = torch.empty((c, plane), device="cuda")
        xd, yd = _lib.cnhw(n, c, h, h, plane), _lib.cnhw(n, c, oh, oh, oplane)
        _lib.call("esgd_maxpool_fwd_f32", y.data_ptr(), yd, 0, am.data_ptr(), x.data_ptr(), xd, 0, k, s, 0, 1,
                  stream_ptr())
        forms = {
            "mask=x": lambda: _lib.call("esgd_maxpool_bwd_f32", dx.data_ptr(), xd, 0, dy.data_ptr(), yd, 0,
                                        am.data_ptr(), x.data_ptr(), 0, k, s, 0, 1, stream_ptr()),
            "gate=y": lambda: _lib.call("esgd_maxpool_bwd_relu_f32", dx.data_ptr(), xd, 0, dy.data_ptr(), yd, 0,
                                        am.data_ptr(), y.data_ptr(), 0, k, s, 0, 1, stream_ptr()),
        }
        for form, fn in forms.items():
            ts = []
            for _ in range(12):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = sorted(ts[2:])[len(ts[2:]) // 2] / 1e3
            alg = 4 * (c * n * oh * oh * 2 + c * n * h * h * (2 if form == "mask=x" else 1)) + 4 * c * n * oh * oh * (
                form == "gate=y")
            print(f"{name} {form}: {t * 1e6:7.1f} us  {alg / t / 1e9:7.0f} GB/s algorithmic ({alg / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
