"""Split-K partials GEMM (pfb_matmul_parts) vs the reduced GEMM (pfb_matmul_ep2),
B pre-split once; device time of 20 replayed launches in a CUDA graph.

    python tools/parts_probe.py [--shape M N K]..."""
import argparse
import ctypes
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1903_04243_b200 import _native as N  # noqa: E402
from paper_1903_04243_b200.executor import DArray  # noqa: E402
from paper_1903_04243_b200.tensor import DType  # noqa: E402


def graph_time(fn, iters=20):
    fn(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for _ in range(iters):
                fn(cs.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    g.replay()
    en.record()
    torch.cuda.synchronize()
    return st.elapsed_time(en) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, action="append")
    ap.add_argument("--force", type=int, default=8)
    args = ap.parse_args()
    lib = N.lib()
    dev = torch.device("cuda")
    for m, n, k in args.shape or [(256, 2048, 1024), (256, 512, 2048), (256, 2048, 512)]:
        a = torch.randn(m, k, device=dev)
        bt = torch.randn(n, k, device=dev) / k ** 0.5
        bias = torch.randn(n, device=dev)
        c = torch.empty(m, n, device=dev)
        A = DArray(a.reshape(-1), 0, a.shape, a.stride(), DType.F64)
        B = DArray(bt.reshape(-1), 0, (k, n), (1, k), DType.F64)
        C = DArray(c.reshape(-1), 0, c.shape, c.stride(), DType.F64)
        X = DArray(bias, 0, (n,), (1,), DType.F64)
        ad, bd, cd, xd = A.desc(), B.desc(), C.desc(), X.desc()
        s = torch.cuda.current_stream().cuda_stream
        pb = torch.empty(lib.pfb_gemm_planes_bytes(bd), dtype=torch.uint8, device=dev)
        lib.pfb_gemm_split_planes(bd, pb.data_ptr(), s)
        need = lib.pfb_matmul_workspace(ad, bd, cd)
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        S = lib.pfb_matmul_parts_count(ad, bd, cd)
        ref = a.double() @ bt.double().t() + bias.double()
        fr = lambda st: lib.pfb_matmul_ep2(ad, bd, cd, None, xd, 0, None, 0, pb.data_ptr(), args.force,
                                           ws.data_ptr(), ws.numel(), st)
        fr(s)
        torch.cuda.synchronize()
        err_red = (c.double() - ref).abs().max().item()
        line = f"{m}x{n}x{k}: "
        if S >= 2:
            parts = torch.empty(S, m, n, device=dev)
            P = DArray(parts.reshape(-1), 0, parts.shape, parts.stride(), DType.F64)
            pd = P.desc()
            fp = lambda st: lib.pfb_matmul_parts(ad, bd, pd, xd, pb.data_ptr(), ws.data_ptr(), ws.numel(), st)
            rc = fp(s)
            torch.cuda.synchronize()
            tot = parts[0].double()
            for j in range(1, S):
                tot = tot + parts[j].double()
            err_p = (tot - ref).abs().max().item()
            tr, tp = [], []
            for _ in range(3):
                tr.append(graph_time(fr))
                tp.append(graph_time(fp))
            line += f"reduced(force {args.force}) {min(tr):6.1f} us (err {err_red:.1e})  parts S={S} rc={rc} {min(tp):6.1f} us (err {err_p:.1e})"
        print(line, flush=True)


if __name__ == "__main__" and "--launches" not in sys.argv:
    main()


def launches_check():
    """kernel launches per pfb_matmul_parts call and the graph period for 1, 5, 20 calls"""
    lib = N.lib()
    dev = torch.device("cuda")
    m, n, k = 256, 2048, 1024
    a = torch.randn(m, k, device=dev)
    bt = torch.randn(n, k, device=dev) / k ** 0.5
    c = torch.empty(m, n, device=dev)
    A = DArray(a.reshape(-1), 0, a.shape, a.stride(), DType.F64)
    B = DArray(bt.reshape(-1), 0, (k, n), (1, k), DType.F64)
    C = DArray(c.reshape(-1), 0, c.shape, c.stride(), DType.F64)
    ad, bd, cd = A.desc(), B.desc(), C.desc()
    s = torch.cuda.current_stream().cuda_stream
    pb = torch.empty(lib.pfb_gemm_planes_bytes(bd), dtype=torch.uint8, device=dev)
    lib.pfb_gemm_split_planes(bd, pb.data_ptr(), s)
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
    S = lib.pfb_matmul_parts_count(ad, bd, cd)
    parts = torch.empty(S, m, n, device=dev)
    pd = DArray(parts.reshape(-1), 0, parts.shape, parts.stride(), DType.F64).desc()
    k0 = lib.pfb_kernel_launches()
    lib.pfb_matmul_parts(ad, bd, pd, None, pb.data_ptr(), ws.data_ptr(), ws.numel(), s)
    print("launches per parts call:", lib.pfb_kernel_launches() - k0)
    for it in (1, 5, 20):
        t = graph_time(lambda st: lib.pfb_matmul_parts(ad, bd, pd, None, pb.data_ptr(), ws.data_ptr(),
                                                       ws.numel(), st), it)
        t2 = graph_time(lambda st: lib.pfb_matmul_ep2(ad, bd, cd, None, None, 0, None, 0, pb.data_ptr(), 0,
                                                      ws.data_ptr(), ws.numel(), st), it)
        print(f"graph of {it}: parts {t:.1f} us/launch, reduced {t2:.1f} us/launch")
    import os
    os.environ["PFB_NO_TMA_STORE"] = "1"


if __name__ == "__main__" and "--launches" in sys.argv:
    launches_check()
