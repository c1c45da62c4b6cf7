"""Host-side tensor values and shape arithmetic.

This module holds *no numeric kernels*: compute happens in the sm_100a
library (`csrc/`).  It provides the value type that crosses the public API
(feeds, constants, results) and the pure shape rules shared by graph
inference and launch-time validation.

Dtype tags follow the reference (`pkg/src/pforvec/tensor.py:28-39`): the
float tag is called ``F64`` for API compatibility, but the B200 path stores and
computes floats in fp32 (BASELINE north_star: fp32 within rtol 1e-4 /
atol 1e-5 of the f64 reference).  ``BOOL`` is stored as one byte.
"""

from __future__ import annotations

import enum

import numpy as np

from .errors import AxisOutOfRange, DuplicateAxis, IncompatibleShapes


class DType(enum.Enum):
    F64 = "f64"
    I64 = "i64"
    BOOL = "bool"

    @property
    def np_dtype(self):
        return {DType.F64: np.float64, DType.I64: np.int64, DType.BOOL: np.bool_}[self]

    @property
    def device_np_dtype(self):
        """numpy dtype of the device representation (fp32 for floats)."""
        return {DType.F64: np.float32, DType.I64: np.int64, DType.BOOL: np.uint8}[self]

    @property
    def itemsize(self) -> int:
        return {DType.F64: 4, DType.I64: 8, DType.BOOL: 1}[self]


def dtype_of_array(arr: np.ndarray) -> DType:
    if arr.dtype == np.bool_:
        return DType.BOOL
    if np.issubdtype(arr.dtype, np.integer):
        return DType.I64
    return DType.F64


class TensorValue:
    """Immutable (by convention) dense host value: a dtype tag + numpy array.

    Float payloads keep whatever float width they were given (f64 constants,
    fp32 device results), so device results are reported at the precision
    they were computed in rather than silently widened.
    """

    __slots__ = ("dtype", "data")

    def __init__(self, dtype: DType, data):
        arr = np.asarray(data)
        if dtype is DType.F64:
            if arr.dtype not in (np.float32, np.float64):
                arr = arr.astype(np.float64)
        else:
            arr = arr.astype(dtype.np_dtype, copy=False)
        if not arr.flags.c_contiguous:
            arr = np.ascontiguousarray(arr)
        self.dtype = dtype
        self.data = arr

    @property
    def shape(self) -> tuple:
        return tuple(self.data.shape)

    @property
    def rank(self) -> int:
        return self.data.ndim

    @property
    def size(self) -> int:
        return int(self.data.size)

    def item(self):
        return self.data.item()

    def __repr__(self):
        return f"TensorValue({self.dtype.value}{list(self.shape)})"


def tensor(values, dtype: DType | None = None) -> TensorValue:
    if isinstance(values, TensorValue):
        if dtype is None or dtype == values.dtype:
            return values
        return TensorValue(dtype, values.data)
    arr = np.asarray(values)
    return TensorValue(dtype if dtype is not None else dtype_of_array(arr), arr)


def scalar(value, dtype: DType | None = None) -> TensorValue:
    return tensor(value, dtype)


def zeros(shape, dtype: DType = DType.F64) -> TensorValue:
    return TensorValue(dtype, np.zeros(tuple(shape), dtype=dtype.np_dtype))


def ones(shape, dtype: DType = DType.F64) -> TensorValue:
    return TensorValue(dtype, np.ones(tuple(shape), dtype=dtype.np_dtype))


def allclose(a: TensorValue, b: TensorValue, tol: float = 1e-9) -> bool:
    """Reference comparator (`tensor.py:419-424`): absolute tol on floats,
    exact equality otherwise."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype == DType.F64:
        return bool(np.allclose(a.data, b.data, rtol=0.0, atol=tol, equal_nan=True))
    return bool(np.array_equal(a.data, b.data))


def parity_close(got: TensorValue, want: TensorValue, rtol=1e-4, atol=1e-5) -> bool:
    """The B200 parity bar: fp32 within rtol/atol of the f64 oracle; ints exact."""
    if got.shape != want.shape or got.dtype != want.dtype:
        return False
    if got.dtype == DType.F64:
        return bool(np.allclose(np.asarray(got.data, np.float64), want.data,
                                rtol=rtol, atol=atol, equal_nan=True))
    return bool(np.array_equal(got.data, want.data))


# --------------------------------------------------------------------------
# shape rules (same semantics as reference tensor.py:104-121, 267-276)

BINARY_OPS = ("add", "sub", "mul", "div", "max", "min", "less", "equal")
COMPARISON_OPS = ("less", "equal")
UNARY_OPS = ("neg", "exp", "log", "relu", "tanh", "sigmoid", "square", "logical_not")
FLOAT_ONLY_UNARY = ("exp", "log", "tanh", "sigmoid")


def broadcast_shapes(a, b) -> tuple:
    """Right-align, then each dim pair must agree or one side must be 1."""
    a, b = tuple(a), tuple(b)
    r = max(len(a), len(b))
    pa = (1,) * (r - len(a)) + a
    pb = (1,) * (r - len(b)) + b
    out = []
    for x, y in zip(pa, pb):
        if x != y and x != 1 and y != 1:
            raise IncompatibleShapes(f"cannot broadcast {pa} with {pb}")
        out.append(y if x == 1 else x)
    return tuple(out)


def normalize_axes(axes, rank: int) -> tuple:
    seen = []
    for ax in axes:
        k = ax + rank if ax < 0 else ax
        if k < 0 or k >= rank:
            raise AxisOutOfRange(f"axis {ax} out of range for rank {rank}")
        seen.append(k)
    if len(set(seen)) != len(seen):
        raise DuplicateAxis(f"duplicate axes after normalization: {axes}")
    return tuple(sorted(seen))


def conv_same_padding(k: int) -> tuple:
    """SAME / stride 1: floor((k-1)/2) before, the remainder after
    (reference tensor.py:209-212)."""
    lo = (k - 1) // 2
    return lo, k - 1 - lo


def resolve_reshape(shape, size: int) -> tuple:
    """Resolve a single -1 wildcard against `size` (reference tensor.py:363-380)."""
    shape = list(shape)
    if shape.count(-1) > 1:
        raise IncompatibleShapes("reshape: more than one -1 dim")
    if -1 in shape:
        known = 1
        for d in shape:
            if d != -1:
                known *= d
        if known == 0:
            shape[shape.index(-1)] = 0
        else:
            if size % known:
                raise IncompatibleShapes(f"reshape: cannot infer -1 in {shape} for size {size}")
            shape[shape.index(-1)] = size // known
    if int(np.prod(shape, dtype=np.int64)) != size:
        raise IncompatibleShapes(f"reshape: target {shape} changes element count {size}")
    return tuple(int(d) for d in shape)
