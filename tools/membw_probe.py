"""Achieved HBM bandwidth of the memory-bound converters at HBM scale
(elementwise / reduction / gather / layout kernels against the
HBM roofline).  Each case is a one-op (or one fused chain) graph on device
constants, executed by the Executor with constant hoisting off and CUDA-graph
replay, so the timed region is exactly that kernel's launch.  Bytes are the
algorithmic ones (distinct inputs read + output written).

    python tools/membw_probe.py [--mb 256] [--peak 6650]
"""
import argparse
import json
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1903_04243_b200 import GraphBuilder  # noqa: E402
from paper_1903_04243_b200.executor import Executor  # noqa: E402
from paper_1903_04243_b200.tensor import DType  # noqa: E402


def timed(graph, reps=20):
    ex = Executor(graph, hoist_constants=False)
    for _ in range(3):
        ex.run_device()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        ex.run_device()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3, ex


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=256, help="size of each fp32 operand in MB")
    ap.add_argument("--peak", type=float, default=6650.0, help="HBM GB/s (MEASURED_PEAKS or fallback)")
    ap.add_argument("--only", default="", help="run only the cases whose name contains this")
    a = ap.parse_args()
    n = a.mb * (1 << 20) // 4
    rows = 16384
    cols = n // rows
    r = np.random.default_rng(0)
    x = r.standard_normal((rows, cols)).astype(np.float32)
    y = r.standard_normal((rows, cols)).astype(np.float32)
    cases = []

    def case(name, build, nbytes):
        if a.only not in name:
            return
        b = GraphBuilder()
        b.graph.set_outputs([build(b)])
        t, ex = timed(b.graph)
        gbs = nbytes / t / 1e9
        cases.append({"case": name, "us": round(t * 1e6, 1), "GB/s": round(gbs), "frac": round(gbs / a.peak, 3),
                      "launches": ex.launch_count})
        print(json.dumps(cases[-1]), flush=True)

    F = 4
    case("binary add [R,C]+[R,C]", lambda b: b.add(b.const(x), b.const(y)), 3 * n * F)
    case("binary mul, stride-0 row broadcast [R,C]*[C]",
         lambda b: b.mul(b.const(x), b.const(y[0])), 2 * n * F + cols * F)
    case("unary tanh", lambda b: b.tanh(b.const(x)), 2 * n * F)
    case("fused chain y*(1-tanh(x)^2)+x (F3)",
         lambda b: b.add(b.mul(b.const(y), b.sub(b.f64(1.0), b.square(b.tanh(b.const(x))))),
                         b.const(x)), 3 * n * F)
    case("reduce_sum rows [R,C]->[R]", lambda b: b.reduce_sum(b.const(x), [1]), n * F + rows * F)
    case("reduce_sum cols [R,C]->[C]", lambda b: b.reduce_sum(b.const(x), [0]), n * F + cols * F)
    idx = r.integers(0, rows, rows).astype(np.int64)
    case("gather_rows [R,C] by random [R] index",
         lambda b: b.gather(b.const(x), b.const(idx, DType.I64)), 2 * n * F + rows * 8)
    case("transpose copy [R,C]->[C,R] (materialised by a reshape)",
         lambda b: b.reshape(b.transpose(b.const(x), [1, 0]), [-1]), 2 * n * F)
    case("tanh of a transposed view", lambda b: b.tanh(b.transpose(b.const(x), [1, 0])), 2 * n * F)
    case("concat [R,C/2]x2 along axis 1",
         lambda b: b.concat([b.const(x[:, :cols // 2]), b.const(x[:, cols // 2:])], 1), 2 * n * F)
    case("cast f32 -> bool (less than 0)", lambda b: b.less(b.const(x), b.f64(0.0)), n * F + n)
    out = pathlib.Path("gpurun_out")
    out.mkdir(exist_ok=True)
    (out / "membw.json").write_text(json.dumps(cases, indent=1))


if __name__ == "__main__":
    main()
