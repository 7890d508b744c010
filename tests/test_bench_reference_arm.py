"""The driver runs `bench.py --impl reference` (the reference's CPU round —
the oracle port — on the host cores); it must work without a GPU and print
one JSON line with the contract's keys."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_contract_line():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--model", "lenet", "--steps", "1",
           "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["model"] == "lenet" and d["higher_is_better"] is True


def test_reference_arm_non_zero_rank_exits_quietly():
    # under torchrun (N > 1) only rank 0 runs the CPU reference and prints
    import os

    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--model", "lenet", "--steps", "1",
           "--warmup", "3", "--gpus", "2"]
    env = dict(os.environ, RANK="1", LOCAL_RANK="1", WORLD_SIZE="2")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
