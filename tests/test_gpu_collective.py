"""The C-ABI collective (include/esgd.h: esgd_nccl_unique_id / esgd_nccl_init
/ esgd_allreduce_sum_f32 / esgd_nccl_destroy) on one GPU: a one-rank
communicator makes the allreduce the identity, which checks the plumbing
(dlopen'ed NCCL, id round trip, stream-ordered call, error mapping). The
two-rank sum is covered by tests/test_gpu_multi.py (path "cabi")."""

import ctypes as C

import pytest
import torch

from paper_1708_02983_b200 import _lib
from paper_1708_02983_b200.device import stream_ptr
from paper_1708_02983_b200.errors import InputError, ShapeError

pytestmark = pytest.mark.gpu


def test_one_rank_allreduce_is_identity():
    lib = _lib.load()
    assert lib.esgd_nccl_available() == 1
    torch.cuda.set_device(0)
    uid = (C.c_ubyte * 128)()
    _lib.check(lib.esgd_nccl_unique_id(C.cast(uid, C.c_void_p)))
    comm = C.c_void_p()
    _lib.check(lib.esgd_nccl_init(C.byref(comm), C.cast(uid, C.c_void_p), 1, 0))
    x = torch.randn(1_000_003, device="cuda")
    ref = x.clone()
    _lib.call("esgd_allreduce_sum_f32", comm, x.data_ptr(), x.numel(), stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    with pytest.raises(ShapeError):
        _lib.call("esgd_allreduce_sum_f32", comm, x.data_ptr(), -1, stream_ptr())
    with pytest.raises(InputError):
        _lib.call("esgd_allreduce_sum_f32", None, x.data_ptr(), 4, stream_ptr())
    _lib.call("esgd_nccl_destroy", comm)


def test_init_rejects_bad_rank():
    uid = (C.c_ubyte * 128)()
    comm = C.c_void_p()
    with pytest.raises(InputError, match="outside world"):
        _lib.check(_lib.load().esgd_nccl_init(C.byref(comm), C.cast(uid, C.c_void_p), 2, 5))
