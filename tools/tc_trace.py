"""Phase timing of one tcgen05 GEMM launch (CTA 0), from globaltimer stamps.

    PFB_TC_TRACE=1 python tools/tc_trace.py --force 4 --shape M N K [--planes] [--graph N]

--planes: B pre-split once (pfb_matmul_ep2, as the executor does for
constant weights).  --graph N: the traced launch is the last of N launches
replayed back to back in a CUDA graph (steady state, programmatic dependent
launch), instead of one launch after an idle gap.  Per k-block (first 16 of
CTA 0): TMA issue, stage landed (split warps), split done, MMA issue."""
import argparse
import ctypes
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1903_04243_b200 import _native as N  # noqa: E402
from paper_1903_04243_b200.executor import DArray  # noqa: E402
from paper_1903_04243_b200.tensor import DType  # noqa: E402

PAIR_NAMES = ["entry", "pdl_done", "tma0_issued", "mma0_issued", "tile0_out", "tile1_out",
              "tile2_out", "tile3_out", "tile4_out", "tile5_out", "tile6_out", "tile7_out", "cta_done"]
PARTS_NAMES = ["entry", "pdl_done", "acc_full", "epilogue_done", "cta_done"]
NAMES = ["entry", "pdl_done", "prologue", "tma0_issued", "stage0_landed", "mma0_issued",
         "last_commit", "acc0_ready", "epilogue_done", "cta_done", "tmem_freed"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", type=int, default=4)
    ap.add_argument("--shape", type=int, nargs="+", required=True)
    ap.add_argument("--planes", action="store_true")
    ap.add_argument("--graph", type=int, default=0)
    ap.add_argument("--parts", action="store_true", help="split-K partials (pfb_matmul_parts)")
    ap.add_argument("--batch", type=int, default=1, help="batched GEMM (the F2 shape: --batch 256)")
    args = ap.parse_args()
    m, n, k = args.shape[:3]
    lib = N.lib()
    lib.pfb_debug_tc_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    dev = torch.device("cuda")
    bs = args.batch
    a = torch.randn(*((bs,) if bs > 1 else ()), m, k, device=dev)
    bt = torch.randn(*((bs,) if bs > 1 else ()), n, k, device=dev)
    c = torch.empty(*((bs,) if bs > 1 else ()), m, n, device=dev)
    A = DArray(a.reshape(-1), 0, a.shape, a.stride(), DType.F64)
    Bt = DArray(bt.reshape(-1), 0, bt.shape, bt.stride(), DType.F64)
    B = Bt.view([k, n], [1, k]) if bs == 1 else Bt.view([bs, k, n], [n * k, 1, k])
    C = DArray(c.reshape(-1), 0, c.shape, c.stride(), DType.F64)
    s = torch.cuda.current_stream().cuda_stream
    ad, bd, cd = A.desc(), B.desc(), C.desc()
    need = lib.pfb_matmul_workspace(ad, bd, cd)
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    planes = None
    if args.planes:
        pb = torch.empty(lib.pfb_gemm_planes_bytes(bd), dtype=torch.uint8, device=dev)
        lib.pfb_gemm_split_planes(bd, pb.data_ptr(), s)
        planes = pb.data_ptr()

    if args.parts:
        S = lib.pfb_matmul_parts_count(ad, bd, cd)
        pt = torch.empty(S, m, n, device=dev)
        pd = DArray(pt.reshape(-1), 0, pt.shape, pt.stride(), DType.F64).desc()

    def call(stream):
        if args.parts:
            return lib.pfb_matmul_parts(pd, bd, pd, None, planes, ws.data_ptr(), ws.numel(), stream) \
                if False else lib.pfb_matmul_parts(ad, bd, pd, None, planes, ws.data_ptr(), ws.numel(), stream)
        if planes is not None:
            return lib.pfb_matmul_ep2(ad, bd, cd, None, None, 0, None, 0, planes, args.force,
                                      ws.data_ptr(), ws.numel(), stream)
        return lib.pfb_matmul_ex(ad, bd, cd, None, 0, args.force, ws.data_ptr(), ws.numel(), stream)

    buf = (ctypes.c_ulonglong * 512)()
    call(s)  # trace buffer allocated outside any capture
    torch.cuda.synchronize()
    for rep in range(3):
        torch.cuda.synchronize()
        if args.graph:
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g, stream=cs):
                    for _ in range(args.graph):
                        rc = call(cs.cuda_stream)
            g.replay()
        else:
            torch.cuda._sleep(1000000)
            rc = call(s)
        torch.cuda.synchronize()
        lib.pfb_debug_tc_trace(buf)
        t0 = buf[0]
        names = PAIR_NAMES if args.force in (5, 6) else NAMES
        if args.parts:
            names = PARTS_NAMES
        print(f"rep {rep} rc={rc}: " + "  ".join(
            f"{nm}={(buf[i] - t0) / 1e3:.2f}" for i, nm in enumerate(names) if buf[i] and buf[i] >= t0))
        st_ = [buf[192 + i] for i in range(160) if buf[192 + i] >= t0]
        en_ = [buf[352 + i] for i in range(160) if buf[352 + i] >= t0]
        if st_ and en_:
            import statistics as S_
            print("   per-CTA start (us): min %.2f med %.2f max %.2f | end: min %.2f med %.2f max %.2f (n=%d)" % (
                (min(st_) - t0) / 1e3, (S_.median(st_) - t0) / 1e3, (max(st_) - t0) / 1e3,
                (min(en_) - t0) / 1e3, (S_.median(en_) - t0) / 1e3, (max(en_) - t0) / 1e3, len(en_)))
        if args.parts:
            print("   kb  tma_issue  landed  mma_issue")
            for kb in range(8):
                v = [buf[16 + kb], buf[48 + kb], buf[32 + kb]]
                if not v[0] or v[0] < t0:
                    break
                print("   %2d  " % kb + "  ".join("%8.2f" % ((x - t0) / 1e3) for x in v))
            continue
        if args.force in (5, 6):
            print("   tile  mma_start  mma_done  drain_start  drained  split_done")
            for t in range(16):
                v = [buf[16 + t], buf[32 + t], buf[48 + t], buf[4 + t] if t < 8 else 0, buf[64 + t]]
                if not v[0] or v[0] < t0:
                    break
                print("   %2d  " % t + "  ".join("%8.2f" % ((x - t0) / 1e3) if x >= t0 else "   -    "
                                                for x in v))
        if args.force not in (5, 6):
            cyc = [buf[96 + kb] for kb in range(16)]
            print("   mma_start deltas (SM cycles):", [int(cyc[i + 1] - cyc[i]) for i in range(15) if cyc[i + 1]])
            print("   kb  tma_issue  landed  split_done  mma_start")
            for kb in range(16):
                v = [buf[16 * j + kb] for j in (1, 2, 3, 4)]
                if not v[0] or v[0] < t0:
                    break
                print("   %2d  " % kb + "  ".join("%8.2f" % ((x - t0) / 1e3) if x >= t0 else "   -    "
                                                 for x in v))


if __name__ == "__main__":
    main()
