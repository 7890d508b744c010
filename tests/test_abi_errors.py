"""C-ABI argument validation (include/esgd.h): every entry point checks its
arguments before touching the device, returns ESGD_ERR_SHAPE / ESGD_ERR_INPUT
with a message in esgd_last_error(), and zero-length work is a no-op — the
reference's ShapeError / InputError contract (updates.py:32-38, 65-68). No
kernel runs here, so these tests need no GPU."""

import ctypes as C

import pytest

from paper_1708_02983_b200 import _lib
from paper_1708_02983_b200.errors import InputError, ShapeError

NULL = None
FAKE = 0x1000  # never dereferenced: validation fails or the size is zero first


def call(name, *args):
    _lib.call(name, *args)


def test_shape_errors_carry_messages():
    with pytest.raises(ShapeError, match="negative"):
        call("esgd_worker_step_f32", FAKE, FAKE, FAKE, FAKE, -1, 0.1, 0.01, NULL)
    with pytest.raises(ShapeError, match="pitch"):
        call("esgd_sync_update_f32", FAKE, 10, FAKE, 10, 2, FAKE, FAKE, 100, 0.1, 0.01, 2, NULL)
    with pytest.raises(ShapeError):
        call("esgd_replica_tree_sum_f32", FAKE, FAKE, 10, 2, 100, NULL)
    with pytest.raises(ShapeError):
        call("esgd_transpose_f32", FAKE, 1, 0, FAKE, 1, 0, -3, 4, 1, NULL)


def test_input_errors():
    with pytest.raises(InputError, match="num_workers"):
        call("esgd_sync_update_f32", FAKE, 64, FAKE, 64, 1, FAKE, FAKE, 64, 0.1, 0.01, 0, NULL)
    with pytest.raises(InputError):  # null buffers with work to do
        call("esgd_worker_step_f32", NULL, FAKE, FAKE, FAKE, 10, 0.1, 0.01, NULL)
    with pytest.raises(InputError, match="batch size"):
        call("esgd_sample_batch_f32", FAKE, 0, FAKE, NULL, FAKE, FAKE, 10, 4, FAKE, FAKE, 11, 1, NULL)
    with pytest.raises(InputError):
        call("esgd_randint_u64", FAKE, 1, 0, 4, 0, NULL)  # upper bound 0
    with pytest.raises(InputError):
        call("esgd_tc_gemm_f32", NULL, NULL)


def test_zero_length_is_a_noop():
    # n = 0: OK without any pointer or launch
    call("esgd_worker_step_f32", NULL, NULL, NULL, NULL, 0, 0.1, 0.01, NULL)
    call("esgd_sync_update_f32", NULL, 0, NULL, 0, 1, NULL, NULL, 0, 0.1, 0.01, 1, NULL)
    call("esgd_measgd_update_f32", NULL, NULL, NULL, NULL, 0, 0.1, 0.9, 0.01, NULL)
    call("esgd_hogwild_apply_f32", NULL, NULL, NULL, 0, 0.01, NULL)


def test_tc_gemm_descriptor_validation():
    d = _lib.TcGemmDesc(64, 64, 32, 1, FAKE, 30, 0, FAKE, 32, 0, FAKE, 64, 1, 0, NULL, 0, NULL, 0, 0, 0, 0, 0, 3,
                        0, 0, NULL, 0)
    with pytest.raises(ShapeError, match="lda"):  # lda < k and not a multiple of 4
        _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), NULL))
    d.lda, d.precision = 32, 2
    with pytest.raises(InputError, match="precision"):
        _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), NULL))
    d.precision, d.act = 3, 7
    with pytest.raises(InputError, match="activation"):
        _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), NULL))
    d.act, d.m = 0, 0  # empty output: no-op
    _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), NULL))


def test_collective_argument_checks():
    # include/esgd.h collective entries: validation before any NCCL call
    with pytest.raises(ShapeError, match="negative"):
        call("esgd_allreduce_sum_f32", NULL, FAKE, -1, NULL)
    call("esgd_allreduce_sum_f32", NULL, NULL, 0, NULL)  # empty: no-op
    with pytest.raises(InputError, match="null"):
        call("esgd_allreduce_sum_f32", NULL, FAKE, 8, NULL)
    comm = C.c_void_p()
    uid = (C.c_ubyte * 128)()
    with pytest.raises(InputError, match="outside world"):
        call("esgd_nccl_init", C.byref(comm), C.cast(uid, C.c_void_p), 2, 2)
    call("esgd_nccl_destroy", NULL)  # null communicator: no-op
    assert _lib.load().esgd_nccl_available() in (0, 1)


def test_round2_entries_validate_before_the_device():
    """the copy-engine round pieces, the SM reserve, the TMA-im2col conv and
    the fused-relu pool backward reject bad arguments without a launch"""
    with pytest.raises(InputError):
        call("esgd_copy_async", NULL, FAKE, 16, NULL)           # null destination with bytes to move
    with pytest.raises(ShapeError):
        call("esgd_copy_async", FAKE, FAKE, -4, NULL)
    call("esgd_copy_async", NULL, NULL, 0, NULL)                # nothing to move: no-op
    with pytest.raises(InputError):
        call("esgd_center_step_sum_f32", FAKE, FAKE, 0, FAKE, 64, 0.01, 2, NULL)    # no sources
    with pytest.raises(InputError):
        call("esgd_center_step_sum_f32", FAKE, FAKE, 9, FAKE, 64, 0.01, 2, NULL)    # > 8 sources
    with pytest.raises(ShapeError):
        call("esgd_center_step_sum_f32", FAKE, FAKE, 2, FAKE, 63, 0.01, 2, NULL)    # not a multiple of 4
    call("esgd_center_step_sum_f32", NULL, NULL, 2, NULL, 0, 0.01, 2, NULL)
    with pytest.raises(InputError):
        call("esgd_set_sm_reserve", -2)
    with pytest.raises(InputError):
        call("esgd_set_sm_reserve", 140)
    call("esgd_set_sm_reserve", 0)
    d = _lib.TcGemmDesc(16, 4, 27, 1, None, 0, 0, FAKE, 28, 0, FAKE, 1, 16, 0, None, 0, None, 0, 0, 0, 0, 0, 3,
                        0, 0, None, 0)
    g = _lib.ConvGather(FAKE, 0, 0, 0, 4, 4, 4, 4, 1, -1, -1, 1, 3, 3, 16, 3)      # 3 channels: not % 32
    assert _lib.load().esgd_tc_conv_tma_f32(C.byref(d), C.byref(g), 1, None) != 0
    with pytest.raises(InputError):
        call("esgd_maxpool_bwd_relu_f32", FAKE, _lib.nchw(1, 1, 4, 4), 0, FAKE, _lib.nchw(1, 1, 2, 2), 0, FAKE,
             NULL, 0, 2, 2, 0, 1, NULL)                           # null pooled output
