"""Every GEMM launch of one AlexNet gradient (production routing), re-run
alone and timed (warm, CUDA events): shape, majors, tile plan, ms, TFLOP/s —
which contractions the round's time goes to.

    python tools/gemm_breakdown.py [--b 128]"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1708_02983_b200 import _lib, network  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402
from paper_1708_02983_b200.nets import DeviceNet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=128)
    ap.add_argument("--model", default="alexnet")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    spec = network.MODELS[a.model](seed=0)
    net = DeviceNet(spec, a.b, 1, torch.device("cuda"))
    W = torch.randn((1, net.ldw), device="cuda") * 0.01
    G = torch.zeros_like(W)
    net.x.normal_()
    net.y.random_(0, spec.num_classes)
    net.gradient(G, W, stream_ptr())
    net.record = []
    net.gradient(G, W, stream_ptr())
    torch.cuda.synchronize()
    recs, net.record = net.record, None
    lib = _lib.load()
    tot = 0.0
    for rec in recs:
        kind, d, fl = rec[0], rec[1], rec[2]
        call = (lambda: lib.esgd_tc_gemm_f32(C.byref(d), stream_ptr())) if kind == "tc" else (
            (lambda: lib.esgd_gemm_f32(C.byref(d), stream_ptr())) if kind == "ffma" else
            (lambda: lib.esgd_tc_conv_f32(C.byref(d), C.byref(rec[3]), rec[4], stream_ptr())))
        for _ in range(2):
            _lib.check(call())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            _lib.check(call())
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / 10
        tot += t
        maj = f"{getattr(d, 'a_major', '-')}{getattr(d, 'b_major', '-')}"
        print(f"{kind:6s} m={d.m:7d} n={d.n:5d} k={d.k:7d} maj={maj} bias={int(bool(d.bias))} mask={int(bool(d.mask))} "
              f"{t:7.3f} ms {fl / t / 1e9:7.1f} TFLOP/s", flush=True)
    print(f"total {tot:.3f} ms over {len(recs)} GEMM launches")


if __name__ == "__main__":
    main()
