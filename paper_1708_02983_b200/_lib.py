"""ctypes binding of libesgd.so (include/esgd.h).

The library is built in-tree (``_build.py``); importing this module never
falls back to anything else: a missing library or a non-sm_100 device raises
``CudaError``. Return codes map onto the reference's exception classes.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import CudaError, InputError, ShapeError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libesgd.so"

OK, ERR_SHAPE, ERR_INPUT, ERR_CUDA, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
ACT = {"none": 0, "relu": 1, "tanh": 2, "sigmoid": 3}

i32, i64, u64, f32, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_void_p


class GemmDesc(C.Structure):
    _fields_ = [
        ("m", i32), ("n", i32), ("k", i32), ("batch", i32),
        ("a", vp), ("a_sm", i64), ("a_sk", i64), ("a_sb", i64),
        ("b", vp), ("b_sk", i64), ("b_sn", i64), ("b_sb", i64),
        ("c", vp), ("c_sm", i64), ("c_sn", i64), ("c_sb", i64),
        ("bias", vp), ("bias_sb", i64),
        ("mask", vp), ("mask_sm", i64), ("mask_sn", i64), ("mask_sb", i64),
        ("c_pre", vp),
        ("act", i32), ("accumulate", i32),
        ("ws", vp), ("ws_floats", i64),
    ]


class TcGemmDesc(C.Structure):
    _fields_ = [
        ("m", i32), ("n", i32), ("k", i32), ("batch", i32),
        ("a", vp), ("lda", i64), ("a_sb", i64),
        ("b", vp), ("ldb", i64), ("b_sb", i64),
        ("c", vp), ("c_sm", i64), ("c_sn", i64), ("c_sb", i64),
        ("bias", vp), ("bias_sb", i64),
        ("mask", vp), ("mask_sm", i64), ("mask_sn", i64), ("mask_sb", i64),
        ("act", i32), ("accumulate", i32), ("precision", i32),
        ("a_major", i32), ("b_major", i32), ("ws", vp), ("ws_floats", i64),
    ]


class ConvGather(C.Structure):
    """esgd_conv_gather (include/esgd.h): the implicitly gathered operand."""
    _fields_ = [
        ("src", vp), ("src_sb", i64), ("plane", i32), ("img_stride", i32), ("src_h", i32), ("src_w", i32),
        ("grid_h", i32), ("grid_w", i32), ("stride", i32), ("yoff", i32), ("xoff", i32), ("sgn", i32),
        ("kh", i32), ("kw", i32), ("npix", i32), ("channels", i32),
    ]


class Tensor4(C.Structure):
    _fields_ = [("n", i32), ("c", i32), ("h", i32), ("w", i32),
                ("sn", i64), ("sc", i64), ("sh", i64), ("sw", i64)]


def nchw(n, c, h, w) -> Tensor4:
    return Tensor4(n, c, h, w, c * h * w, h * w, w, 1)


def nhwc(n, c, h, w) -> Tensor4:
    return Tensor4(n, c, h, w, h * w * c, 1, w * c, c)


def cnhw(n, c, h, w, plane_pitch: int) -> Tensor4:
    """channel-major over the batch: element (img, ci, y, x) at
    ci*plane_pitch + (img*h + y)*w + x, plane_pitch >= n*h*w."""
    return Tensor4(n, c, h, w, h * w, plane_pitch, w, 1)


_SIGS = {
    "esgd_last_error": (C.c_char_p, []),
    "esgd_abi_version": (C.c_int, []),
    "esgd_device_ok": (C.c_int, [C.c_int]),
    "esgd_worker_step_f32": (C.c_int, [vp, vp, vp, vp, i64, f32, f32, vp]),
    "esgd_center_step_from_sum_f32": (C.c_int, [vp, vp, vp, i64, f32, i32, vp]),
    "esgd_sync_update_f32": (C.c_int, [vp, i64, vp, i64, i32, vp, vp, i64, f32, f32, i32, vp]),
    "esgd_sync_update_nvls_f32": (C.c_int, [vp, i64, vp, i64, i32, vp, vp, vp, vp, i64, i32, i32, f32, f32, i32,
                                            vp]),
    "esgd_nvls_barrier": (C.c_int, [vp, i32, i32, vp, vp]),
    "esgd_nccl_available": (C.c_int, []),
    "esgd_nccl_unique_id": (C.c_int, [vp]),
    "esgd_nccl_init": (C.c_int, [vp, vp, i32, i32]),
    "esgd_allreduce_sum_f32": (C.c_int, [vp, vp, i64, vp]),
    "esgd_nccl_destroy": (C.c_int, [vp]),
    "esgd_center_step_nvls_f32": (C.c_int, [vp, vp, vp, i64, i32, i32, f32, i32, i32, vp]),
    "esgd_worker_step_sum_f32": (C.c_int, [vp, i64, vp, i64, i32, vp, vp, i64, f32, f32, vp]),
    "esgd_sync_update_sum_f32": (C.c_int, [vp, i64, vp, i64, i32, vp, vp, vp, i64, f32, f32, i32, vp]),
    "esgd_measgd_update_f32": (C.c_int, [vp, vp, vp, vp, i64, f32, f32, f32, vp]),
    "esgd_center_step_snapshots_f32": (C.c_int, [vp, vp, vp, i64, i32, i64, f32, vp]),
    "esgd_sync_update_solo_f32": (C.c_int, [vp, vp, vp, i64, f32, f32, vp]),
    "esgd_center_incr_f32": (C.c_int, [vp, vp, vp, i64, f32, vp]),
    "esgd_exchange_update_f32": (C.c_int, [vp, vp, vp, i64, f32, f32, vp]),
    "esgd_sgd_step_f32": (C.c_int, [vp, vp, i64, f32, vp]),
    "esgd_msgd_step_f32": (C.c_int, [vp, vp, vp, i64, f32, f32, vp]),
    "esgd_hogwild_apply_f32": (C.c_int, [vp, vp, vp, i64, f32, vp]),
    "esgd_hogwild_axpy_f32": (C.c_int, [vp, vp, i64, f32, vp]),
    "esgd_replica_tree_sum_f32": (C.c_int, [vp, vp, i64, i32, i64, vp]),
    "esgd_randint_u64": (C.c_int, [vp, u64, u64, i64, u64, vp]),
    "esgd_sample_batch_f32": (C.c_int, [vp, i64, vp, vp, vp, vp, i64, i64, vp, vp, i32, i32, vp]),
    "esgd_gather_rows_h2d": (C.c_int, [vp, i64, vp, i64, vp, i32, i64, i64, vp]),
    "esgd_quadratic_grad_f32": (C.c_int, [vp, i64, vp, i64, i32, vp, vp, i64, vp]),
    "esgd_gemm_f32": (C.c_int, [C.POINTER(GemmDesc), vp]),
    "esgd_tc_gemm_f32": (C.c_int, [C.POINTER(TcGemmDesc), vp]),
    "esgd_gemm_ws_floats": (C.c_int, [C.POINTER(GemmDesc), C.POINTER(i64)]),
    "esgd_async_ctl_ints": (C.c_int, [i32]),
    "esgd_async_preload": (C.c_int, []),
    "esgd_enable_peer_access": (C.c_int, [i32, i32]),
    "esgd_async_master_f32": (C.c_int, [vp, i64, vp, vp, vp, i32, i64, f32, i32, vp]),
    "esgd_async_post": (C.c_int, [vp, i32, i32, vp, vp]),
    "esgd_async_wait": (C.c_int, [vp, i32, i32, vp, vp]),
    "esgd_tc_conv_f32": (C.c_int, [C.POINTER(TcGemmDesc), C.POINTER(ConvGather), i32, vp]),
    "esgd_tc_conv_tma_f32": (C.c_int, [C.POINTER(TcGemmDesc), C.POINTER(ConvGather), i32, vp]),
    "esgd_set_sm_reserve": (C.c_int, [i32]),
    "esgd_center_step_sum_f32": (C.c_int, [vp, vp, i32, vp, i64, f32, i32, vp]),
    "esgd_copy_async": (C.c_int, [vp, vp, i64, vp]),
    "esgd_tc_conv_ws_floats": (C.c_int, [C.POINTER(TcGemmDesc), C.POINTER(i64)]),
    "esgd_tc_gemm_ws_floats": (C.c_int, [C.POINTER(TcGemmDesc), C.POINTER(i64)]),
    "esgd_act_fwd_f32": (C.c_int, [vp, vp, i64, i32, vp]),
    "esgd_act_bwd_f32": (C.c_int, [vp, vp, i64, i32, vp]),
    "esgd_softmax_xent_f32": (C.c_int, [vp, vp, vp, i64, i64, vp, i64, i32, i32, i32, vp, vp]),
    "esgd_transpose_f32": (C.c_int, [vp, i64, i64, vp, i64, i64, i32, i32, i32, vp]),
    "esgd_argmax_rows_f32": (C.c_int, [vp, vp, i64, i32, i32, vp]),
    "esgd_colsum_f32": (C.c_int, [vp, i64, vp, i64, i64, i64, i32, i32, vp, vp]),
    "esgd_im2col_f32": (C.c_int, [vp, i64, i64, i64, vp, Tensor4, i64, i32, i32, i32, i32, i32, i32, i32, vp]),
    "esgd_col2im_f32": (C.c_int, [vp, Tensor4, i64, vp, i64, i64, i64, i32, i32, i32, i32, i32, i32, vp, i64, i32, vp]),
    "esgd_rowsum_f32": (C.c_int, [vp, i64, vp, i64, i64, i32, i64, i32, vp, vp]),
    "esgd_maxpool_fwd_f32": (C.c_int, [vp, Tensor4, i64, vp, vp, Tensor4, i64, i32, i32, i32, i32, vp]),
    "esgd_maxpool_bwd_f32": (C.c_int, [vp, Tensor4, i64, vp, Tensor4, i64, vp, vp, i64, i32, i32, i32, i32, vp]),
    "esgd_maxpool_bwd_relu_f32": (C.c_int, [vp, Tensor4, i64, vp, Tensor4, i64, vp, vp, i64, i32, i32, i32, i32, vp]),
    "esgd_copy4_f32": (C.c_int, [vp, Tensor4, i64, vp, Tensor4, i64, i32, vp]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building if needed) libesgd.so; raises CudaError if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    override = os.environ.get("ESGD_LIB")  # experiments: load a prebuilt variant, never rebuild
    if override:
        build_if_missing = False
    if build_if_missing:
        try:
            from . import _build
            _build.build()
        except Exception as exc:  # no nvcc on the box: use the shipped .so
            if not LIB_PATH.exists():
                raise CudaError(f"libesgd.so missing and cannot be built: {exc}") from exc
    path = Path(override) if override else LIB_PATH
    if not path.exists():
        raise CudaError(f"libesgd.so not found at {path}")
    lib = C.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().esgd_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = last_error()
    if rc == ERR_SHAPE:
        raise ShapeError(msg)
    if rc == ERR_INPUT:
        raise InputError(msg)
    raise CudaError(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
