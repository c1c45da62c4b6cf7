"""GPU: the conv kernels against the oracle (f64 restatement of reference
tensor.py:209-260) -- the per-example tiled conv2d, and the fused filter
gradient conv_filter_grad (im2col(x_b)^T gy_b without the im2col buffer)
including shapes that take the im2col + GEMM fallback.  Bar: rtol 1e-4 /
atol 1e-5."""

import numpy as np
import pytest

from oracle import kernels as K
from paper_1903_04243_b200 import GraphBuilder
from paper_1903_04243_b200.tensor import DType, TensorValue

pytestmark = pytest.mark.gpu

SHAPES = [  # n, h, w, c, o, k1, k2
    (5, 28, 28, 1, 8, 3, 3),     # cfg2 ConvNet (tiled)
    (3, 6, 6, 1, 4, 5, 5),       # 5x5 window (tiled)
    (2, 9, 7, 3, 5, 3, 3),       # no tiled kernel: im2col + GEMM / direct
    (4, 5, 8, 3, 8, 3, 3),       # KC = 27 (tiled forward)
    (1, 1, 1, 1, 1, 3, 3),       # 1x1 image: all taps but the centre in the halo
]


@pytest.fixture(scope="module")
def Executor():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1903_04243_b200.executor import Executor
    return Executor


def _f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


@pytest.mark.parametrize("shape", SHAPES)
def test_conv_filter_grad(shape, Executor):
    n, h, w, c, o, k1, k2 = shape
    r = np.random.default_rng(sum(shape))
    x, gy = _f32(r.standard_normal((n, h, w, c))), _f32(r.standard_normal((n, h, w, o)))
    b = GraphBuilder()
    node = b.graph.add_node("conv_filter_grad", [(b.const(x).nid, 0), (b.const(gy).nid, 0)],
                            {"k1": k1, "k2": k2})
    b.graph.set_outputs([b.graph.out(node.id)])
    (got,) = Executor(b.graph, optimize=False).run()
    want = K.conv_filter_grad(TensorValue(DType.F64, x), TensorValue(DType.F64, gy), k1, k2).data
    np.testing.assert_allclose(np.asarray(got.data, np.float64), want, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("shape", SHAPES)
def test_conv2d_forward(shape, Executor):
    n, h, w, c, o, k1, k2 = shape
    r = np.random.default_rng(sum(shape) + 1)
    x, f = _f32(r.standard_normal((n, h, w, c))), _f32(r.standard_normal((k1, k2, c, o)))
    b = GraphBuilder()
    b.graph.set_outputs([b.conv2d(b.const(x), b.const(f))])
    (got,) = Executor(b.graph, optimize=False).run()
    want = K.conv2d(TensorValue(DType.F64, x), TensorValue(DType.F64, f)).data
    np.testing.assert_allclose(np.asarray(got.data, np.float64), want, rtol=1e-4, atol=1e-5)


def test_cfg2_conv_has_no_im2col_buffer(Executor):
    """The optimised cfg2 ConvNet program computes its filter gradients with
    conv_filter_grad: no im2col kernel runs."""
    from paper_1903_04243_b200 import workloads as WL
    w = WL.cfg2(WL.this_api(), n=8, model="conv")
    ex = Executor(w.graph)
    ex.kernel_timer = []
    ex.run(feeds=w.feeds)
    kinds = {r[0] for r in ex.kernel_timer}
    assert "conv_filter_grad" in kinds and "im2col" not in kinds
