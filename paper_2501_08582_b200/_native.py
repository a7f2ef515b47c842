"""ctypes binding of the C ABI in include/lors_b200.h.

The shared library is built in-tree (paper_2501_08582_b200/_native/liblors_b200.so
by `build.py`).  There is no CPU fallback: if the library is missing or the
device is not sm_100, every call raises DeviceError.
"""

from __future__ import annotations

import ctypes as ct
import os
import threading

from .errors import ArgumentError, DeviceError, ShapeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_native", "liblors_b200.so")
# tools/ kernel experiments load alternative builds of the same sources
LIB_PATH = os.environ.get("LORS_B200_LIB", LIB_PATH)

LORS_OK, LORS_ERR_SHAPE, LORS_ERR_ARGUMENT, LORS_ERR_DEVICE, LORS_ERR_CUDA = range(5)
DTYPE_F32, DTYPE_BF16 = 0, 1
MASK_FROM_W, MASK_BITS = 0, 1
GRAD_STE, GRAD_MASKED = 0, 1
FLAG_EMIT_P = 1 << 0
FLAG_SPARSE24 = 1 << 1
FLAG_NO_DX = 1 << 2
FLAG_DX_ONLY = 1 << 3
FLAG_ZEROED = 1 << 4
FLAG_DETERMINISTIC = 1 << 5
FLAG_NO_TAIL_SPLIT = 1 << 6
FLAG_FAULT_DA_SIGN = 1 << 30

# Every symbol include/lors_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED_SYMBOLS = (
    "lors_fwd", "lors_fwd_workspace", "lors_fwd_group", "lors_fwd_group_workspace", "lors_bwd", "lors_bwd_workspace",
    "lors_effective_weight", "lors_pack_mask", "lors_compress_24", "lors_grad_outer",
    "lors_last_error", "lors_abi_version", "lors_device_check",
    "lors_launch_count", "lors_reset_launch_count",
)
# include/lors_decoder.h: decoder-side helpers (not the LoRS drop-in boundary)
DECODER_SYMBOLS = ("lors_rope", "lors_swiglu", "lors_swiglu_bwd", "lors_add3", "lors_add_rmsnorm", "lors_add_rmsnorm_bwd",
                   "lors_cross_entropy", "lors_cross_entropy_bwd", "lors_adamw", "lors_adamw_dstep",
                   "lors_adamw_p2p")

_vp = ct.c_void_p


class FwdArgs(ct.Structure):
    _fields_ = [
        ("L", ct.c_int64), ("R", ct.c_int64), ("C", ct.c_int64), ("r", ct.c_int64),
        ("dtype", ct.c_int32), ("mask_mode", ct.c_int32), ("flags", ct.c_uint32),
        ("alpha", ct.c_float),
        ("x", _vp), ("w", _vp), ("mask_bits", _vp), ("w24", _vp), ("meta24", _vp),
        ("a", _vp), ("b", _vp), ("bias", _vp), ("y", _vp), ("p", _vp),
        ("workspace", _vp), ("workspace_bytes", ct.c_size_t),
    ]


class BwdArgs(ct.Structure):
    _fields_ = [
        ("L", ct.c_int64), ("R", ct.c_int64), ("C", ct.c_int64), ("r", ct.c_int64),
        ("dtype", ct.c_int32), ("mask_mode", ct.c_int32), ("grad_mode", ct.c_int32),
        ("flags", ct.c_uint32), ("alpha", ct.c_float),
        ("x", _vp), ("w", _vp), ("mask_bits", _vp), ("a", _vp), ("b", _vp), ("dy", _vp),
        ("p", _vp), ("dx", _vp), ("da", _vp), ("db", _vp), ("dbias", _vp),
        ("workspace", _vp), ("workspace_bytes", ct.c_size_t),
    ]


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ct.CDLL:
    """Load (once) and type the native library; raises DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"native library {path} is missing; run `python -m paper_2501_08582_b200.build` "
                "(there is no CPU fallback)")
        lib = ct.CDLL(path)
        lib.lors_fwd.argtypes = [ct.POINTER(FwdArgs), _vp]
        lib.lors_fwd.restype = ct.c_int
        lib.lors_fwd_workspace.argtypes = [ct.POINTER(FwdArgs)]
        lib.lors_fwd_workspace.restype = ct.c_size_t
        lib.lors_fwd_group.argtypes = [ct.POINTER(FwdArgs), ct.c_int32, _vp]
        lib.lors_fwd_group.restype = ct.c_int
        lib.lors_fwd_group_workspace.argtypes = [ct.POINTER(FwdArgs), ct.c_int32]
        lib.lors_fwd_group_workspace.restype = ct.c_size_t
        lib.lors_bwd.argtypes = [ct.POINTER(BwdArgs), _vp]
        lib.lors_bwd.restype = ct.c_int
        lib.lors_bwd_workspace.argtypes = [ct.POINTER(BwdArgs)]
        lib.lors_bwd_workspace.restype = ct.c_size_t
        lib.lors_effective_weight.argtypes = [ct.c_int64, ct.c_int64, ct.c_int64, ct.c_int32, ct.c_int32,
                                              ct.c_float, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.lors_effective_weight.restype = ct.c_int
        lib.lors_pack_mask.argtypes = [ct.c_int64, ct.c_int64, ct.c_int32, _vp, _vp, _vp]
        lib.lors_pack_mask.restype = ct.c_int
        lib.lors_compress_24.argtypes = [ct.c_int64, ct.c_int64, ct.c_int32, _vp, _vp, _vp, _vp, _vp]
        lib.lors_compress_24.restype = ct.c_int
        lib.lors_grad_outer.argtypes = [ct.c_int64, ct.c_int64, ct.c_int64, ct.c_int32, ct.c_int32,
                                        _vp, _vp, _vp, _vp, _vp]
        lib.lors_grad_outer.restype = ct.c_int
        lib.lors_last_error.argtypes = []
        lib.lors_last_error.restype = ct.c_char_p
        lib.lors_abi_version.restype = ct.c_int
        lib.lors_device_check.restype = ct.c_int
        lib.lors_rope.argtypes = [_vp, _vp, _vp, _vp, ct.c_int64, ct.c_int64, ct.c_int64, ct.c_int64, ct.c_int32,
                                  ct.c_int32, _vp]
        lib.lors_rope.restype = ct.c_int
        lib.lors_swiglu.argtypes = [_vp, _vp, _vp, ct.c_int64, _vp]
        lib.lors_swiglu.restype = ct.c_int
        lib.lors_swiglu_bwd.argtypes = [_vp, _vp, _vp, _vp, _vp, ct.c_int64, _vp]
        lib.lors_swiglu_bwd.restype = ct.c_int
        lib.lors_add3.argtypes = [_vp, _vp, _vp, _vp, ct.c_int64, _vp]
        lib.lors_add3.restype = ct.c_int
        lib.lors_add_rmsnorm.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ct.c_int64, ct.c_int64, ct.c_float, _vp]
        lib.lors_add_rmsnorm.restype = ct.c_int
        lib.lors_add_rmsnorm_bwd.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ct.c_int64, ct.c_int64, _vp]
        lib.lors_add_rmsnorm_bwd.restype = ct.c_int
        lib.lors_cross_entropy.argtypes = [_vp, _vp, _vp, _vp, ct.c_int64, ct.c_int64, _vp]
        lib.lors_cross_entropy.restype = ct.c_int
        lib.lors_cross_entropy_bwd.argtypes = [_vp, _vp, _vp, _vp, _vp, ct.c_int64, ct.c_int64, _vp]
        lib.lors_cross_entropy_bwd.restype = ct.c_int
        lib.lors_adamw.argtypes = [_vp, _vp, _vp, _vp, _vp, ct.c_int64, ct.c_float, ct.c_float, ct.c_float,
                                   ct.c_float, ct.c_float, ct.c_int64, _vp]
        lib.lors_adamw.restype = ct.c_int
        lib.lors_adamw_dstep.argtypes = [_vp, _vp, _vp, _vp, _vp, ct.c_int64, ct.c_float, ct.c_float, ct.c_float,
                                         ct.c_float, ct.c_float, _vp, _vp]
        lib.lors_adamw_dstep.restype = ct.c_int
        lib.lors_adamw_p2p.argtypes = [_vp, _vp, _vp, _vp, _vp, ct.c_int64, ct.c_int32, ct.c_int32, ct.c_float,
                                       ct.c_float, ct.c_float, ct.c_float, ct.c_float, ct.c_int64, _vp]
        lib.lors_adamw_p2p.restype = ct.c_int
        lib.lors_launch_count.restype = ct.c_uint64
        lib.lors_reset_launch_count.restype = None
        _lib = lib
        return lib


def check(status: int) -> None:
    """Raise the reference-vocabulary exception for a non-OK status."""
    if status == LORS_OK:
        return
    msg = load().lors_last_error().decode(errors="replace")
    if status == LORS_ERR_SHAPE:
        raise ShapeError(msg)
    if status == LORS_ERR_ARGUMENT:
        raise ArgumentError(msg)
    raise DeviceError(f"lors native status {status}: {msg}")


def launch_count() -> int:
    return int(load().lors_launch_count())


def reset_launch_count() -> None:
    load().lors_reset_launch_count()
