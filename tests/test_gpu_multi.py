"""Multi-GPU Sync EASGD (one process per GPU, NCCL allreduce captured in the
round's CUDA graph) — runs only where >= 2 GPUs are visible; equality with
the single-process run is bitwise at N = 2 (tools/dist_check.py)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("path", ["nvls", "ce", "ce1", "nccl", "cabi"])
def test_two_rank_sync_easgd_equals_single_process(path):
    """NVLS-fused round update (multimem ld_reduce / st over NVSwitch), its
    copy-engine variant (peer slices moved by cudaMemcpyAsync; "ce1": one
    worker per rank, peers read each other's W in place), the
    torch.distributed NCCL allreduce, and the allreduce through libesgd's own
    NCCL communicator (esgd_allreduce_sum_f32) all equal the single-process
    run bit for bit."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", str(ROOT / "tools" / "dist_check.py")]
    env = dict(os.environ, ESGD_NVLS={"nvls": "1", "ce": "ce", "ce1": "ce"}.get(path, "0"))
    if path == "ce1":
        env["DIST_PER_RANK"] = "1"
    if path == "cabi":
        env["ESGD_COLLECTIVE"] = "cabi"
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert "DIST_CHECK PASS" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    if path in ("cabi", "ce", "ce1"):
        assert f"collective={'nccl-cabi' if path == 'cabi' else 'nvls-ce'}" in r.stdout, r.stdout[-2000:]
    print(r.stdout[-400:])
