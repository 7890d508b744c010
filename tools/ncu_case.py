"""Small, deterministic launch sequences for ncu captures (profiles/).

    python tools/ncu_case.py update     # fused elastic update on 61.1M params (AlexNet size), 5 launches
    python tools/ncu_case.py update_sum # the same + next round's replica sum (the engine's round update)
    python tools/ncu_case.py dgrad      # tcgen05 conv2 dgrad GEMM (M=93312 N=1600 K=192), 4 launches
    python tools/ncu_case.py fwd        # tcgen05 conv2 forward GEMM (M=93312 N=192 K=1600), 4 launches
    python tools/ncu_case.py wgrad      # tcgen05 conv2 wgrad GEMM (M=192 N=1600 K=93312), 4 launches
    python tools/ncu_case.py im2col     # AlexNet conv2 im2col (64x27x27 -> colT[1600][93312]), 4 launches
    python tools/ncu_case.py im2col1    # AlexNet conv1 im2col (3x224x224, 11x11 s4 -> colT[363][387200])
    python tools/ncu_case.py col2im     # AlexNet conv2 col2im (colT[1600][93312] -> 64x27x27), 4 launches
    python tools/ncu_case.py poolbwd    # AlexNet pool1 backward (64x55x55 <- 64x27x27, 3/2), 4 launches
"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200 import HyperParams, _lib  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402
from paper_1708_02983_b200.updates import sync_update_, sync_update_sum_  # noqa: E402


def update_solo():
    """the P = 1 round update (esgd_sync_update_solo_f32), 61.1M params"""
    from paper_1708_02983_b200.updates import sync_update_solo_
    n = 61_100_840
    ld = (n + 63) // 64 * 64
    W = torch.randn((1, ld), device="cuda")
    G = torch.randn_like(W)
    Cc = torch.randn(ld, device="cuda")
    hy = HyperParams(eta=0.01, rho=0.1)
    for _ in range(5):
        sync_update_solo_(W, G, Cc, n, hy)
    torch.cuda.synchronize()


def update(fused=False):
    n = 61_100_840
    ld = (n + 63) // 64 * 64
    W = torch.randn((1, ld), device="cuda")
    G = torch.randn_like(W)
    Cc = torch.randn(ld, device="cuda")
    S = torch.randn(ld, device="cuda")
    hy = HyperParams(eta=0.01, rho=0.1)
    for _ in range(5):
        if fused:
            sync_update_sum_(W, G, Cc, S, S, n, 8, hy)
        else:
            sync_update_(W, G, Cc, S, n, 8, hy)
    torch.cuda.synchronize()


def gemm(m, n, k, am, bm, cm):
    kp, mp, np_ = (k + 3) // 4 * 4, (m + 3) // 4 * 4, (n + 3) // 4 * 4
    A = torch.randn(kp * mp, device="cuda")
    B = torch.randn(kp * np_, device="cuda")
    Cm = torch.empty(mp * np_, device="cuda")
    ws = torch.zeros(1 << 24, device="cuda")
    c_sm, c_sn = (1, mp) if cm else (np_, 1)
    d = _lib.TcGemmDesc(m, n, k, 1, A.data_ptr(), mp if am else kp, 0, B.data_ptr(), np_ if bm else kp, 0,
                        Cm.data_ptr(), c_sm, c_sn, 0, None, 0, None, 0, 0, 0, 0, 0, 3, am, bm,
                        ws.data_ptr(), ws.numel())
    for _ in range(4):
        _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
    torch.cuda.synchronize()


def im2col(c, h, k, stride, pad, back=False):
    b = 128
    oh = (h + 2 * pad - k) // stride + 1
    npix = b * oh * oh
    np4 = (npix + 3) // 4 * 4
    kd = c * k * k
    x = torch.randn(c * b * h * h, device="cuda")
    col = torch.randn(kd * np4, device="cuda")
    xd = _lib.cnhw(b, c, h, h, b * h * h)
    lib = _lib.load()
    for _ in range(4):
        if back:
            _lib.check(lib.esgd_col2im_f32(x.data_ptr(), xd, 0, col.data_ptr(), 1, np4, 0, k, k, stride, pad,
                                           oh, oh, None, 0, 1, stream_ptr()))
        else:
            _lib.check(lib.esgd_im2col_f32(col.data_ptr(), 1, np4, 0, x.data_ptr(), xd, 0, k, k, stride, pad,
                                           oh, oh, 1, stream_ptr()))
    torch.cuda.synchronize()


def poolbwd():
    b, c, h = 128, 64, 55
    oh = (h - 3) // 2 + 1
    x = torch.randn(c * b * h * h, device="cuda")
    y = torch.empty(c * b * oh * oh, device="cuda")
    am = torch.empty(c * b * oh * oh, dtype=torch.int32, device="cuda")
    xd, yd = _lib.cnhw(b, c, h, h, b * h * h), _lib.cnhw(b, c, oh, oh, b * oh * oh)
    lib = _lib.load()
    _lib.check(lib.esgd_maxpool_fwd_f32(y.data_ptr(), yd, 0, am.data_ptr(), x.data_ptr(), xd, 0, 3, 2, 0, 1,
                                        stream_ptr()))
    for _ in range(4):
        _lib.check(lib.esgd_maxpool_bwd_f32(x.data_ptr(), xd, 0, y.data_ptr(), yd, 0, am.data_ptr(), None, 0,
                                            3, 2, 0, 1, stream_ptr()))
    torch.cuda.synchronize()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    case = sys.argv[1]
    if case == "update":
        update()
    elif case == "update_solo":
        update_solo()
    elif case == "update_sum":
        update(fused=True)
    elif case == "dgrad":
        gemm(93312, 1600, 192, 1, 0, 1)
    elif case == "fwd":
        gemm(93312, 192, 1600, 1, 0, 1)
    elif case == "wgrad":
        gemm(192, 1600, 93312, 0, 0, 0)
    elif case == "im2col":
        im2col(64, 27, 5, 1, 2)
    elif case == "im2col1":
        im2col(3, 224, 11, 4, 2)
    elif case == "col2im":
        im2col(64, 27, 5, 1, 2, back=True)
    elif case == "poolbwd":
        poolbwd()
    print("ok", case)
