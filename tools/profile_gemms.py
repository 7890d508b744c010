"""Time every GEMM of one gradient pass on its own (warm, CUDA events).

    python tools/profile_gemms.py --model lenet
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1708_02983_b200 import HyperParams, _lib, make_config, network  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402
from paper_1708_02983_b200.trainers.synchronous import SyncEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="lenet")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    wl = bench.WORKLOADS[args.model]
    spec = network.MODELS[args.model](seed=0)
    train, _ = bench.make_data(args.model, spec)
    prob = NetworkProblem(spec, train)
    cfg = make_config("sync-easgd3", workers=1, iterations=5, batch_size=wl["b"],
                      hyper=HyperParams(eta=wl["eta"], rho=wl["rho"]), seed=3)
    eng = SyncEngine(cfg, prob, use_graph=False, profile_rounds=0)
    net = eng.plan.net
    net.record = []
    eng.plan.gradient(eng.G, eng.W, stream_ptr())
    torch.cuda.synchronize()
    lib = _lib.load()
    tot = 0.0
    for kind, d, fl in net.record:
        fn = lib.esgd_tc_gemm_f32 if kind == "tc" else lib.esgd_gemm_f32
        for _ in range(3):
            _lib.check(fn(C.byref(d), stream_ptr()))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            _lib.check(fn(C.byref(d), stream_ptr()))
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) / 20
        tot += t
        print(f"{kind:4s} m={d.m:7d} n={d.n:5d} k={d.k:7d} batch={d.batch}  {t * 1e3:8.1f} us  {fl / t / 1e9:7.2f} TFLOP/s")
    print(f"total {tot * 1e3:.1f} us")


if __name__ == "__main__":
    main()
