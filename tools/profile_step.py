"""Per-kernel GPU time of Sync-EASGD rounds (CUPTI via torch.profiler; warm
caches, graph replays) — the optimisation loop's view; ncu gives the cold,
serialised launch list for profiles/.

    python tools/profile_step.py --model lenet --steps 20
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1708_02983_b200 import HyperParams, make_config, network  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402
from paper_1708_02983_b200.trainers.synchronous import SyncEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="lenet")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--graph", type=int, default=1)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    wl = bench.WORKLOADS[args.model]
    b = args.batch or wl["b"]
    spec = network.MODELS[args.model](seed=0)
    train, _ = bench.make_data(args.model, spec)
    prob = NetworkProblem(spec, train)
    cfg = make_config("sync-easgd3", workers=args.workers, iterations=args.steps + 5, batch_size=b,
                      hyper=HyperParams(eta=wl["eta"], rho=wl["rho"]), seed=3)
    eng = SyncEngine(cfg, prob, use_graph=bool(args.graph), profile_rounds=2)
    for _ in range(5):
        eng.step()
    torch.cuda.synchronize()
    net = eng.plan.net
    print(f"GEMM routing per round: tcgen05={net.tc_calls // 6} ffma={net.ffma_calls // 6}")
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        eng.step()
    t1.record()
    t1.synchronize()
    step_ms = t0.elapsed_time(t1) / args.steps
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            eng.step()
        torch.cuda.synchronize()
    rows = []
    for e in prof.key_averages():
        dev_us = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
        if dev_us > 0:
            rows.append((dev_us / args.steps, e.count // args.steps, e.key[:90]))
    rows.sort(reverse=True)
    tot = sum(r[0] for r in rows)
    print(f"step {step_ms * 1e3:.1f} us (events); kernel sum {tot:.1f} us/step")
    for us, cnt, name in rows[:30]:
        print(f"{us:9.1f} us/step  x{cnt:<3d} {100 * us / tot:5.1f}%  {name}")


if __name__ == "__main__":
    main()
