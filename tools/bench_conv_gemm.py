"""Implicit-GEMM convolutions (esgd_tc_conv_f32) on AlexNet b=128 layer
shapes: forward, weight gradient, data gradient (CUDA events, warm).

    python tools/bench_conv_gemm.py [--b 128] [--only conv2] [--tma]
Reports ms and fp32-equivalent TFLOP/s (2*M*N*K / t). --tma: the TMA
im2col-mode variant (esgd_tc_conv_tma_f32, NHWC sources, K = (kh, kw, c)),
plus the CNHW -> NHWC transposes it needs (esgd_transpose_f32)."""

import argparse
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200 import _lib  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402

LAYERS = [("conv1", 3, 224, 64, 11, 4, 2), ("conv2", 64, 27, 192, 5, 1, 2), ("conv3", 192, 13, 384, 3, 1, 1),
          ("conv4", 384, 13, 256, 3, 1, 1), ("conv5", 256, 13, 256, 3, 1, 1)]


def r4(x):
    return (x + 3) // 4 * 4


TMA = False


def timed_fn(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def timed(d, g, side, reps=10):
    lib = _lib.load()
    need = C.c_int64(0)
    _lib.check(lib.esgd_tc_conv_ws_floats(C.byref(d), C.byref(need)))
    ws = torch.zeros(max(4, need.value), device="cuda")
    d.ws, d.ws_floats = ws.data_ptr(), ws.numel()
    fn = lib.esgd_tc_conv_tma_f32 if TMA else lib.esgd_tc_conv_f32
    return timed_fn(lambda: _lib.check(fn(C.byref(d), C.byref(g), side, stream_ptr())), reps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=128)
    ap.add_argument("--only", default="")
    ap.add_argument("--pass", dest="which", default="", help="fwd | wgrad | dgrad (default all)")
    ap.add_argument("--tma", action="store_true")
    a = ap.parse_args()
    global TMA
    TMA = a.tma
    n = a.b
    tot = 0.0
    for name, cin, h, cout, k, s, p in LAYERS:
        if a.only and a.only != name:
            continue
        oh = (h + 2 * p - k) // s + 1
        K = cin * k * k
        xplane, oplane = r4(n * h * h), r4(n * oh * oh)
        X = torch.randn(cin * xplane, device="cuda")
        D = torch.randn(cout * oplane, device="cuda")
        W = torch.randn(cout * r4(K), device="cuda")
        Wp = torch.randn(cin * r4(cout * k * k), device="cuda")
        out = torch.empty(cout * oplane, device="cuda")
        dW = torch.empty(cout * K, device="cuda")
        dx = torch.empty(cin * xplane, device="cuda")
        bias = torch.randn(cout, device="cuda")
        npo, npi = n * oh * oh, n * h * h
        if TMA and cin % 32:
            continue
        if TMA:  # NHWC copies of the input and of the output gradient
            Xn = torch.empty(npi * cin, device="cuda")
            Dn = torch.empty(npo * cout, device="cuda")
            lib = _lib.load()
            tx = timed_fn(lambda: _lib.check(lib.esgd_transpose_f32(Xn.data_ptr(), cin, 0, X.data_ptr(), xplane, 0,
                                                                    cin, npi, 1, stream_ptr())))
            td = timed_fn(lambda: _lib.check(lib.esgd_transpose_f32(Dn.data_ptr(), cout, 0, D.data_ptr(), oplane, 0,
                                                                    cout, npo, 1, stream_ptr())))
            print(f"{name}.nhwc  x {tx * 1e3:8.3f} ms  delta {td * 1e3:8.3f} ms", flush=True)
            tot += tx + td
            gx = _lib.ConvGather(Xn.data_ptr(), 0, 0, 0, h, h, oh, oh, s, -p, -p, 1, k, k, npo, cin)
        else:
            gx = _lib.ConvGather(X.data_ptr(), 0, xplane, 0, h, h, oh, oh, s, -p, -p, 1, k, k, npo, cin)
        d = _lib.TcGemmDesc(npo, cout, K, 1, None, 0, 0, W.data_ptr(), r4(K), 0, out.data_ptr(), 1, oplane, 0,
                            bias.data_ptr(), 0, None, 0, 0, 0, 1, 0, 3, 0, 0, None, 0)
        want = lambda kind: not a.which or a.which == kind
        rows = [("fwd", timed(d, gx, 1), 2.0 * npo * cout * K)] if want("fwd") else []
        d = _lib.TcGemmDesc(cout, K, npo, 1, D.data_ptr(), oplane, 0, None, 0, 0, dW.data_ptr(), K, 1, 0,
                            None, 0, None, 0, 0, 0, 0, 0, 3, 0, 0, None, 0)
        if want("wgrad"):
            rows.append(("wgrad", timed(d, gx, 2), 2.0 * npo * cout * K))
        if s == 1 and name != "conv1" and want("dgrad"):
            kd = cout * k * k
            if TMA:
                q = k - 1 - p
                gd = _lib.ConvGather(Dn.data_ptr(), 0, 0, 0, oh, oh, h, h, 1, -q, -q, 1, k, k, npi, cout)
            else:
                gd = _lib.ConvGather(D.data_ptr(), 0, oplane, 0, oh, oh, h, h, 1, p, p, -1, k, k, npi, cout)
            d = _lib.TcGemmDesc(npi, cin, kd, 1, None, 0, 0, Wp.data_ptr(), r4(kd), 0, dx.data_ptr(), 1, xplane, 0,
                                None, 0, X.data_ptr(), 1, xplane, 0, 0, 0, 3, 0, 0, None, 0)
            rows.append(("dgrad", timed(d, gd, 1), 2.0 * npi * cin * kd))
        for kind, t, fl in rows:
            tot += t
            print(f"{name}.{kind:5s} {t * 1e3:8.3f} ms  {fl / t / 1e12:7.1f} TFLOP/s fp32-eq  "
                  f"{3 * fl / t / 1e12:7.1f} tf32-pipe", flush=True)
    print(f"total {tot * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
