"""Probe the symmetric-memory / multicast plumbing of the NVLS round update:

    torchrun --nproc-per-node 2 tools/probe_nvls.py
"""
import os
import sys
import traceback
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    import torch.distributed._symmetric_memory as symm
    try:
        print(rank, "backend", symm.get_backend(torch.device("cuda", local)) if hasattr(symm, "get_backend") else "?")
    except Exception as e:
        print(rank, "get_backend failed", e)
    try:
        from paper_1708_02983_b200.fabric.nvls import NvlsRound
        r = NvlsRound(1024, torch.device("cuda", local))
        print(rank, "NVLS OK mc", hex(r.mc), "flags", r.peer_flags.tolist())
        S = r.S[0]
        S.fill_(rank + 1.0)
        torch.cuda.synchronize()
        dist.barrier()
        # one round through the fused kernel: W/G zeros, C[0] = 0 -> C[1] = er * sum(S)
        from paper_1708_02983_b200 import HyperParams
        W = torch.zeros((1, 1024), device="cuda")
        G = torch.zeros_like(W)
        hy = HyperParams(eta=0.5, rho=0.5)
        r.update(W, G, 0, 2, hy)
        torch.cuda.synchronize()
        dist.barrier()
        print(rank, "C[1][:4] =", r.C[1][:4].tolist(), "expected", hy.etarho32 * 3.0)
    except Exception:
        traceback.print_exc()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
