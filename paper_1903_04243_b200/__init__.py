"""B200-native execution of statically vectorized parallel-for (arXiv 1903.04243).

Drop-in for the reference `pforvec` hot path: the same graph-building API
(`GraphBuilder`, `pfor`, `jacobian`, `per_example_gradients`, `map_fn`, plus
`vectorized_map` and `batch_jacobian`), with `Executor` running every
converted op as a hand-written sm_100a kernel behind the C ABI in
`include/pfb.h`.  There is no CPU fallback: without the built library or a
CUDA device, `Executor` raises `errors.NativeUnavailable`.
"""

from . import errors
from .apps import batch_jacobian, jacobian, map_fn, per_example_gradients, pfor, vectorized_map
from .autodiff import gradient
from .builder import GraphBuilder
from .graph import Block, Graph, Node, Ref
from .tensor import DType, TensorValue, allclose, ones, parity_close, scalar, tensor, zeros
from .vectorize import (Diagnostics, Policy, WrappedValue, b200_registry, default_registry,
                        reference_registry, vectorize_body, vectorize_graph)

__version__ = "0.1.0"


def __getattr__(name):
    # the device runtime imports torch; keep graph construction import-light
    if name in ("Executor", "execute", "RngState", "VariableStore"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)


__all__ = [
    "Block", "DType", "Diagnostics", "Executor", "Graph", "GraphBuilder", "Node", "Policy",
    "Ref", "RngState", "TensorValue", "VariableStore", "WrappedValue", "allclose",
    "b200_registry", "batch_jacobian", "default_registry", "errors", "execute", "gradient",
    "jacobian", "map_fn", "ones", "parity_close", "per_example_gradients", "pfor",
    "reference_registry", "scalar", "tensor", "vectorize_body", "vectorize_graph",
    "vectorized_map", "zeros",
]
