"""Single-op graphs for the golden kernel cases (tests/golden/make_golden.py).

`build_case(name, ins)` returns a graph (this package's IR) whose one output
is the op the golden case recorded from the reference kernel, so the same
case runs through the oracle (CPU tests) and the device executor (GPU tests).
"""

import numpy as np

from paper_1903_04243_b200 import DType, GraphBuilder

IM2COL_K = {0: (3, 3), 1: (3, 3), 2: (2, 4)}
REDUCE_AXES = {0: (1,), 1: (0, 2), 2: (-1,), 3: (0, 1), 4: (1,), 5: (0,), 6: (1, 3)}


def case_names(kernels):
    return sorted({k.split("/")[0] for k in kernels if k.endswith("/out")})


def inputs(kernels, name):
    pre = f"{name}/in/"
    return {k[len(pre):]: v for k, v in kernels.items() if k.startswith(pre)}


def _c(b, v):
    v = np.asarray(v)
    if v.dtype == np.float32:
        v = v.astype(np.float64)
    return b.const(v)


def build_case(name, ins):
    b = GraphBuilder()
    parts = name.split("_")
    if parts[0] == "binary":
        op = parts[1]
        out = b._add(op, [_c(b, ins["a"]), _c(b, ins["b"])])
    elif parts[0] == "unary":
        op = "logical_not" if name.startswith("unary_logical_not") else parts[1]
        out = b._add(op, [_c(b, ins["x"])])
    elif parts[0] == "cast":
        dt = {"i": DType.I64, "b": DType.BOOL, "f": DType.F64}[parts[2]]
        out = b.cast(_c(b, ins["x"]), dt)
    elif parts[0] == "matmul":
        out = b.matmul(_c(b, ins["a"]), _c(b, ins["b"]))
    elif name.startswith("conv2d_input_grad"):
        out = b.conv2d_input_grad(_c(b, ins["gy"]), _c(b, ins["f"]))
    elif parts[0] == "conv2d":
        out = b.conv2d(_c(b, ins["x"]), _c(b, ins["f"]))
    elif parts[0] == "im2col":
        k1, k2 = IM2COL_K[int(parts[1])]
        out = b.im2col(_c(b, ins["x"]), k1, k2)
    elif name == "reduce_sum_i64":
        out = b.reduce_sum(_c(b, ins["x"]), (0,))
    elif parts[0] == "reduce":
        out = b.reduce_sum(_c(b, ins["x"]), REDUCE_AXES[int(parts[2])])
    elif name == "concat_ax1":
        out = b.concat([_c(b, ins["a"]), _c(b, ins["b"])], 1)
    elif name == "concat_ax0":
        out = b.concat([_c(b, ins["a"]), _c(b, ins["b"])], 0)
    elif parts[0] == "gather":
        out = b.gather(_c(b, ins["x"]), _c(b, ins["i"]))
    elif name == "scatter_rows":
        out = b.scatter_rows([_c(b, ins["i0"]), _c(b, ins["i1"])],
                             [_c(b, ins["p0"]), _c(b, ins["p1"])], b.i64(6))
    elif name == "scatter_add_dup":
        out = b.scatter_add_rows(_c(b, ins["i"]), _c(b, ins["u"]), 5)
    elif name == "scatter_add_scalar":
        out = b.scatter_add_rows(_c(b, ins["i"]), _c(b, ins["u"]), 4)
    elif name == "transpose":
        out = b.transpose(_c(b, ins["x"]), (2, 0, 1))
    elif name == "stack":
        out = b.stack([_c(b, ins["a"]), _c(b, ins["b"])])
    elif name == "tile_leading":
        out = b.tile_leading(_c(b, ins["x"]), b.i64(3))
    elif name == "slice_leading":
        out = b.slice_leading(_c(b, ins["x"]), b.i64(2))
    elif name == "where_true":
        out = b.where_true(_c(b, ins["m"]))
    elif name == "complement":
        out = b.complement(_c(b, ins["idx"]), b.i64(int(ins["total"])))
    elif name == "rng":
        out = None  # needs an RngState; handled by the callers
    else:
        raise KeyError(name)
    if out is not None:
        b.graph.set_outputs([out])
    return b.graph
