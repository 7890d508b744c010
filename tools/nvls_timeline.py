"""Timeline of the overlapped multi-GPU round (sync-easgd3) per rank: the
forward/backward on the compute stream and the collective (NVLS center or
NCCL allreduce) on the comm stream, from CUDA events of eager rounds.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nvls_timeline.py [--rounds 5]
Prints per rank and round: forward/backward ms, collective start / end
relative to the round start, and the exposed wait at the join."""
import argparse
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_1708_02983_b200 import HyperParams, make_config, network  # noqa: E402
from paper_1708_02983_b200.trainers import NetworkProblem  # noqa: E402
from paper_1708_02983_b200.trainers.synchronous import SyncEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--model", default="alexnet")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    wl = bench.WORKLOADS[a.model]
    spec = network.MODELS[a.model](seed=0)
    train, test = bench.make_data(a.model, spec)
    prob = NetworkProblem(spec, train, test)
    cfg = make_config("sync-easgd3", workers=world, iterations=a.rounds + 2, batch_size=wl["b"],
                      hyper=HyperParams(eta=wl["eta"], rho=wl["rho"]), seed=3)
    eng = SyncEngine(cfg, prob, use_graph=False, profile_rounds=0)
    eng.step()
    eng.step()
    torch.cuda.synchronize()
    names = ("t0", "c0", "c1", "g1", "j", "u1")
    for r in range(a.rounds):
        dist.barrier()
        ev = {k: torch.cuda.Event(enable_timing=True) for k in names}
        eng.step_eager(ev)
        eng.advance()
        ev["u1"].synchronize()
        t = lambda k: ev["t0"].elapsed_time(ev[k])
        print(f"rank {rank} round {r}: fwd/bwd {t('g1'):.3f} ms | comm {t('c0'):.3f} -> {t('c1'):.3f} ms "
              f"({t('c1') - t('c0'):.3f}) | join wait {t('j') - t('g1'):.3f} | update {t('u1') - t('j'):.3f} | "
              f"round {t('u1'):.3f} [{eng.collective}]", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
