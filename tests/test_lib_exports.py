"""The C-ABI library loads without a GPU and exports exactly what
include/esgd.h declares (no compute calls here)."""

import ctypes
import re
from pathlib import Path

from paper_1708_02983_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared():
    text = (ROOT / "include" / "esgd.h").read_text()
    return sorted(set(re.findall(r"\b(esgd_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    raw = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared():
        assert hasattr(raw, name), name
    assert lib.esgd_abi_version() == 1


def test_argument_validation_without_gpu():
    lib = _lib.load()
    # shape / domain errors are detected on the host before any launch
    assert lib.esgd_center_step_from_sum_f32(None, None, None, 10, 0.1, 0, None) == _lib.ERR_INPUT
    assert "num_workers" in _lib.last_error()
    assert lib.esgd_worker_step_f32(None, None, None, None, -1, 0.1, 0.1, None) == _lib.ERR_SHAPE
    assert lib.esgd_randint_u64(None, 1, 0, 4, 0, None) == _lib.ERR_INPUT
    assert lib.esgd_replica_tree_sum_f32(None, None, 0, 65, 8, None) == _lib.ERR_UNSUPPORTED


def test_no_b200_reports_cleanly():
    import torch
    if torch.cuda.is_available():
        return
    assert _lib.load().esgd_device_ok(0) == 0
    assert _lib.last_error()


def test_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
