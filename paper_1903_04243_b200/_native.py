"""ctypes binding of libpfb.so (the C ABI declared in include/pfb.h).

The shared library is built in-tree (`csrc/Makefile`, or
`__graft_entry__.build()`) and loaded from this package directory.  If it is
missing, or no CUDA device is visible, `lib()` raises NativeUnavailable: the
executor has no CPU fallback by design.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

from .errors import NativeUnavailable

MAX_RANK = 8
LIB_PATH = pathlib.Path(__file__).with_name("libpfb.so")

F32, I64, BOOL = 0, 1, 2
BINARY_CODES = {"add": 0, "sub": 1, "mul": 2, "div": 3, "max": 4, "min": 5, "less": 6, "equal": 7}
UNARY_CODES = {"neg": 0, "exp": 1, "log": 2, "relu": 3, "tanh": 4, "sigmoid": 5, "square": 6,
               "logical_not": 7}
DEV_OOB, DEV_COLLISION, DEV_COVER = 1, 2, 4
E_DTYPE, E_SHAPE, E_RANK, E_ARG, E_UNSUPPORTED = 1, 2, 3, 4, 5


class PfbTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p),
                ("dtype", ctypes.c_int32),
                ("rank", ctypes.c_int32),
                ("shape", ctypes.c_int64 * MAX_RANK),
                ("stride", ctypes.c_int64 * MAX_RANK)]


_P = ctypes.POINTER(PfbTensor)
_vp, _i32, _i64, _u32, _u64, _f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double)

_SIGNATURES = {
    "pfb_version": ([], ctypes.c_int),
    "pfb_device_sm_count": ([], ctypes.c_int),
    "pfb_binary": ([_i32, _P, _P, _P, _vp], ctypes.c_int),
    "pfb_unary": ([_i32, _P, _P, _vp], ctypes.c_int),
    "pfb_cast": ([_P, _P, _vp], ctypes.c_int),
    "pfb_fused_ew": ([_i32, _P, _i32, ctypes.POINTER(_i32), _P, _vp], ctypes.c_int),
    "pfb_fused_ew_multi": ([_i32, _P, _i32, ctypes.POINTER(_i32), _i32, ctypes.POINTER(_i32), _P,
                            _vp], ctypes.c_int),
    "pfb_fused_ew_parts": ([_i32, _P, ctypes.POINTER(ctypes.c_int64), _i32, ctypes.POINTER(_i32),
                            _i32, ctypes.POINTER(_i32), _P, _vp], ctypes.c_int),
    "pfb_fused_ew_rows": ([_i32, _P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_i32), _i32,
                           ctypes.POINTER(_i32), _i32, ctypes.POINTER(_i32), _P, _vp], ctypes.c_int),
    "pfb_fused_parts_ok": ([], ctypes.c_int),
    "pfb_col_dots": ([_i32, _P, _P, _P, _vp], ctypes.c_int),
    "pfb_row_sum_parts": ([_P, _i32, ctypes.c_int64, _P, _vp], ctypes.c_int),
    "pfb_fused_jit_config": ([_i32, ctypes.c_int64], ctypes.c_int),
    "pfb_kernel_launches": ([], ctypes.c_int64),
    "pfb_fused_jit_check": ([_i32, _i32, ctypes.c_uint64, _i32, ctypes.POINTER(_i32), _i32, ctypes.POINTER(_i32),
                             _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32)], ctypes.c_int),
    "pfb_fused_int": ([_i32, _P, _i32, ctypes.POINTER(_i32), _i32, ctypes.POINTER(_i32), _P,
                       _vp], ctypes.c_int),
    "pfb_reduce_dot": ([_P, _P, _u32, _P, _vp, _i64, _vp], ctypes.c_int),
    "pfb_select": ([_P, _P, _P, _P, _vp], ctypes.c_int),
    "pfb_reduce_sum": ([_P, _u32, _P, _vp, _i64, _vp], ctypes.c_int),
    "pfb_copy": ([_P, _P, _vp], ctypes.c_int),
    "pfb_copy_many": ([_i32, _P, _P, _vp], ctypes.c_int),
    "pfb_pack": ([_i32, _P, _vp, ctypes.POINTER(_i64), _vp], ctypes.c_int),
    "pfb_fill": ([_P, _f64, _vp], ctypes.c_int),
    "pfb_matmul_workspace": ([_P, _P, _P], ctypes.c_int64),
    "pfb_matmul": ([_P, _P, _P, _vp, _i64, _vp], ctypes.c_int),
    "pfb_matmul_ex": ([_P, _P, _P, _vp, _i32, _i32, _vp, _i64, _vp], ctypes.c_int),
    "pfb_matmul_ep": ([_P, _P, _P, _P, _P, _i32, _P, _i32, _vp, _i32, _i32, _vp, _i64, _vp],
                      ctypes.c_int),
    "pfb_matmul_dual_workspace": ([_P, _P, _P, _P, _P], ctypes.c_int64),
    "pfb_gemm_planes_bytes": ([_P], ctypes.c_int64),
    "pfb_conv2d_filter_grad": ([_P, _P, _i32, _i32, _P, _P, _vp], ctypes.c_int),
    "pfb_gemm_split_planes": ([_P, _vp, _vp], ctypes.c_int),
    "pfb_matmul_ep2": ([_P, _P, _P, _P, _P, _i32, _P, _i32, _vp, _i32, _vp, _i64, _vp],
                       ctypes.c_int),
    "pfb_matmul_parts_count": ([_P, _P, _P], ctypes.c_int),
    "pfb_matmul_parts_workspace": ([_P, _P, _P], ctypes.c_int64),
    "pfb_matmul_parts": ([_P, _P, _P, _P, _vp, _vp, _i64, _vp], ctypes.c_int),
    "pfb_matmul_dual_parts_count": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "pfb_matmul_dual_parts_workspace": ([_P, _P, _P, _P, _P], ctypes.c_int64),
    "pfb_matmul_dual_parts": ([_P, _P, _P, _P, _P, _P, _vp, _vp, _vp, _i64, _vp], ctypes.c_int),
    "pfb_matmul_dual2": ([_P, _P, _P, _P, _P, _P, _i32, _vp, _vp, _i32, _vp, _i64, _vp],
                         ctypes.c_int),
    "pfb_matmul_dual": ([_P, _P, _P, _P, _P, _P, _i32, _i32, _vp, _i64, _vp], ctypes.c_int),
    "pfb_concat": ([_i32, _P, _i32, _P, _vp], ctypes.c_int),
    "pfb_loop_create": ([ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_uint64)],
                        ctypes.c_int),
    "pfb_set_condition": ([ctypes.c_uint64, _vp, _vp, _vp], ctypes.c_int),
    "pfb_set_condition_any": ([ctypes.c_uint64, _vp, ctypes.c_int64, _vp, _vp], ctypes.c_int),
    "pfb_copy_many_cond": ([_i32, _P, _P, _i32, ctypes.c_uint64, _vp, _vp, _vp], ctypes.c_int),
    "pfb_loop_finalize": ([_vp, _vp, _vp], ctypes.c_int),
    "pfb_loop_launch": ([_vp, _vp], ctypes.c_int),
    "pfb_loop_destroy": ([_vp], ctypes.c_int),
    "pfb_row_dots": ([_i32, _P, _P, _P, _vp], ctypes.c_int),
    "pfb_matmul_fused": ([_P, _P, _P, _P, _P, _i32, _vp, _i32, _i32, _vp, _i64, _vp], ctypes.c_int),
    "pfb_im2col": ([_P, _i32, _i32, _P, _vp], ctypes.c_int),
    "pfb_conv2d": ([_P, _P, _P, _vp], ctypes.c_int),
    "pfb_conv2d_input_grad": ([_P, _P, _P, _vp], ctypes.c_int),
    "pfb_gather_rows": ([_P, _P, _P, _vp, _vp], ctypes.c_int),
    "pfb_gather_stacked": ([_P, _P, _P, _vp, _vp], ctypes.c_int),
    "pfb_gather_stacked_many": ([_P, _i32, _P, _P, _vp, _vp], ctypes.c_int),
    "pfb_scatter_rows": ([_i32, _P, _P, _i64, _P, _vp, _vp, _vp], ctypes.c_int),
    "pfb_scatter_add_rows": ([_P, _P, _i64, _P, _vp, _vp], ctypes.c_int),
    "pfb_where_true": ([_P, _P, _vp, _vp, _i64, _vp], ctypes.c_int),
    "pfb_complement": ([_P, _i64, _P, _vp, _vp, _i64, _vp], ctypes.c_int),
    "pfb_iota": ([_P, _i64, _vp], ctypes.c_int),
    "pfb_rng_uniform": ([_u64, _u64, _P, _vp], ctypes.c_int),
    "pfb_outer_sq_norm": ([_P, _P, _P, _vp], ctypes.c_int),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load(path=None, require_device=False):
    """Load the shared library (no GPU needed just to load and inspect it)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = pathlib.Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(f"{p} not built; run `make -C {p.parent / 'csrc'}` "
                                "or __graft_entry__.build()")
    try:
        handle = ctypes.CDLL(str(p), mode=os.RTLD_LOCAL)
    except OSError as e:
        raise NativeUnavailable(f"cannot load {p}: {e}") from e
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = handle
    return handle


def lib():
    """The library, with a CUDA device required (the product path)."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the pfor executor has no CPU fallback")
    return load()
