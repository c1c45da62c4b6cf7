"""Phase timing of one tcgen05 GEMM launch (CTA 0), from globaltimer stamps.

    PFB_TC_TRACE=1 python tools/tc_trace.py --force 4 --shape M N K [B]
"""
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
NAMES = ["entry", "pdl_done", "prologue", "tma0_issued", "stage0_landed", "mma0_issued",
         "last_commit", "acc0_ready", "epilogue_done", "cta_done", "tmem_freed"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", type=int, default=4)
    ap.add_argument("--shape", type=int, nargs="+", required=True)
    args = ap.parse_args()
    m, n, k = args.shape[:3]
    lib = N.lib()
    lib.pfb_debug_tc_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    dev = torch.device("cuda")
    a = torch.randn(m, k, device=dev)
    bt = torch.randn(n, k, device=dev)
    c = torch.empty(m, n, device=dev)
    A = DArray(a.reshape(-1), 0, a.shape, a.stride(), DType.F64)
    Bt = DArray(bt.reshape(-1), 0, bt.shape, bt.stride(), DType.F64)
    B = Bt.view([k, n], [1, k])
    C = DArray(c.reshape(-1), 0, c.shape, c.stride(), DType.F64)
    s = torch.cuda.current_stream().cuda_stream
    need = lib.pfb_matmul_workspace(A.desc(), B.desc(), C.desc())
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    buf = (ctypes.c_ulonglong * 16)()
    for rep in range(4):
        torch.cuda.synchronize()
        torch.cuda._sleep(1000000)
        rc = lib.pfb_matmul_ex(A.desc(), B.desc(), C.desc(), None, 0, args.force, ws.data_ptr(),
                               ws.numel(), s)
        torch.cuda.synchronize()
        lib.pfb_debug_tc_trace(buf)
        t0 = buf[0]
        names = PAIR_NAMES if args.force in (5, 6) else NAMES
        print(f"rep {rep} rc={rc}: " + "  ".join(
            f"{nm}={(buf[i] - t0) / 1e3:.2f}" for i, nm in enumerate(names) if buf[i] and buf[i] >= t0))


if __name__ == "__main__":
    main()
