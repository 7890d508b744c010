"""Recalibrate the alpha-beta cost model on B200:

    torchrun --nproc-per-node N tools/calibrate_costmodel.py

Times ncclAllReduce of 4 KB .. 256 MB payloads (CUDA events, max over
ranks), fits alpha/beta, measures the AlexNet round's forward/backward on
the device, and prints the predicted Sync-EASGD round at N = 1..1024.
"""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200.fabric import costmodel  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cm, samples = costmodel.calibrate_allreduce()
    if dist.get_rank() == 0:
        world = dist.get_world_size()
        out = {"world": world, "alpha_s": cm.alpha, "beta_s_per_byte": cm.beta,
               "bus_GBps_equiv": (2 * (world - 1) / world) / cm.beta / 1e9 if cm.beta else None,
               "samples": [{"bytes": b, "seconds": t, "algbw_GBps": b / t / 1e9} for b, t in samples]}
        # AlexNet: 61.1M params; compute/update from bench (4.4 ms fwd+bwd, 0.28 ms update at N=1)
        out["predict_alexnet"] = {n: costmodel.predict_sync_round(cm, 4.4e-3, 61_100_840, n, 0.28e-3, 0.4)
                                  for n in (1, 2, 4, 8, 72, 1024)}
        print(json.dumps(out, indent=1))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
