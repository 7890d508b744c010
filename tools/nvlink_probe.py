"""Which NVLink traffic counters this driver exposes (NVML field values,
nvidia-smi nvlink -gt d), read around a 1 GiB NCCL allreduce on 2 GPUs:
    torchrun --nproc-per-node 2 tools/nvlink_probe.py"""
import os
import subprocess

import pynvml as N
import torch
import torch.distributed as dist

rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(rank)
names = [x for x in dir(N) if x.startswith("NVML_FI_DEV_NVLINK") and ("BYTES" in x or "THROUGHPUT" in x or "PACKETS" in x)]


def read():
    out = {}
    for nm in names:
        fid = getattr(N, nm)
        tot, rcs = 0, set()
        for link in list(range(18)) + [0xFFFFFFFF]:
            try:
                v = N.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                rcs.add(v.nvmlReturn)
                if v.nvmlReturn == 0:
                    tot += int(v.value.ullVal) if link != 0xFFFFFFFF else 0
            except Exception as e:
                rcs.add(str(e)[:30])
        out[nm] = (tot, sorted(map(str, rcs)))
    return out


x = torch.ones(256 << 20, device="cuda")
a = read()
if rank == 0:
    s0 = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout
for _ in range(4):
    dist.all_reduce(x)
torch.cuda.synchronize()
b = read()
if rank == 0:
    s1 = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout
    for k in names:
        print(k, b[k][0] - a[k][0], a[k][1])
    print("smi before:\n", s0[:600], "\nsmi after:\n", s1[:600])
dist.barrier()
