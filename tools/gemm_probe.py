"""Time the GEMM paths on representative shapes (CUDA events, device time).

    python tools/gemm_probe.py [--force 2] [--shape M N K [B]] [--iters 20]
"""
import argparse
import sys
import pathlib

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1903_04243_b200 import _native as N  # noqa: E402
from paper_1903_04243_b200.executor import DArray  # noqa: E402
from paper_1903_04243_b200.tensor import DType  # noqa: E402

GRAPH = False
PLANES = False
SHAPES = [(10240, 784, 256, 1), (256, 1024, 2048, 1), (256, 2048, 1024, 1),
          (4096, 4096, 4096, 1), (1024, 2048, 64, 64)]


def run(lib, m, n, k, bsz, force, iters):
    dev = torch.device("cuda")
    a = torch.randn(bsz, m, k, device=dev) if bsz > 1 else torch.randn(m, k, device=dev)
    bt = torch.randn(bsz, n, k, device=dev) / k ** 0.5 if bsz > 1 else torch.randn(n, k, device=dev) / k ** 0.5
    c = torch.empty(*(a.shape[:-1] + (n,)), device=dev)
    A = DArray(a.reshape(-1), 0, a.shape, a.stride(), DType.F64)
    Bt = DArray(bt.reshape(-1), 0, bt.shape, bt.stride(), DType.F64)
    perm = list(range(bt.dim()))
    perm[-1], perm[-2] = perm[-2], perm[-1]
    B = Bt.view([Bt.shape[p] for p in perm], [Bt.strides[p] for p in perm])
    C = DArray(c.reshape(-1), 0, c.shape, c.stride(), DType.F64)
    s = torch.cuda.current_stream().cuda_stream
    ad, bd, cd = A.desc(), B.desc(), C.desc()
    need = lib.pfb_matmul_workspace(ad, bd, cd)
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    wp, wn = ws.data_ptr(), ws.numel()
    planes = None
    if PLANES:  # B's hi/lo planes made once (a loop-invariant weight)
        pb = torch.empty(lib.pfb_gemm_planes_bytes(bd), dtype=torch.uint8, device=dev)
        lib.pfb_gemm_split_planes(bd, pb.data_ptr(), s)
        planes = pb.data_ptr()

    def call(stream):
        if planes is not None:
            return lib.pfb_matmul_ep2(ad, bd, cd, None, None, 0, None, 0, planes, force, wp, wn,
                                      stream)
        return lib.pfb_matmul_ex(ad, bd, cd, None, 0, force, wp, wn, stream)

    for _ in range(3):
        rc = call(s)
        if rc != 0:
            raise RuntimeError(f"matmul returned {rc}")
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GRAPH:
        # device time without host launch overhead: replay a captured graph
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                for _ in range(iters):
                    call(cs.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        st.record()
        g.replay()
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / iters
        flops = 2.0 * bsz * m * n * k
        ref = (a.double() @ bt.double().transpose(-1, -2))
        err = (c.double() - ref).abs().max().item()
        return ms, flops / ms / 1e9, err
    torch.cuda._sleep(int(20e6))
    st.record()
    for _ in range(iters):
        call(s)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / iters
    flops = 2.0 * bsz * m * n * k
    ref = (a.double() @ bt.double().transpose(-1, -2))
    err = (c.double() - ref).abs().max().item()
    return ms, flops / ms / 1e9, err


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", type=int, default=2)
    ap.add_argument("--shape", type=int, nargs="+")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--graph", action="store_true", help="time a replayed CUDA graph")
    ap.add_argument("--planes", action="store_true", help="B pre-split once (pfb_matmul_ep2)")
    args = ap.parse_args()
    global GRAPH, PLANES
    GRAPH = args.graph
    PLANES = args.planes
    lib = N.lib()
    shapes = [tuple(args.shape) + ((1,) if len(args.shape) == 3 else ())] if args.shape else SHAPES
    for shp in shapes:
        ms, tf, err = run(lib, *shp, args.force, args.iters)
        print(f"force={args.force} MxNxK(xB)={shp}: {ms*1e3:9.1f} us  {tf:8.1f} TFLOP/s  maxerr {err:.2e}",
              flush=True)


if __name__ == "__main__":
    main()
