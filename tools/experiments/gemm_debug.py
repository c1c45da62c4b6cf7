"""Bring-up check of the tcgen05 operand feeds: every operand layout x feed
(3 = pre-split, 4 = raw TMA) against f64 numpy; prints max error per case."""
import sys
import pathlib

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_1903_04243_b200 import _native as N  # noqa: E402
from paper_1903_04243_b200.executor import DArray  # noqa: E402
from paper_1903_04243_b200.tensor import DType  # noqa: E402
import test_gpu_gemm as T  # noqa: E402

env = (torch, N.lib(), DArray, DType)
shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or \
    [(128, 128, 32), (128, 128, 64), (256, 2048, 1024), (200, 300, 100)]
for shp in shapes:
    m, n, k = shp
    r = np.random.default_rng(0)
    a, b = T._operands(r, (m, k), (k, n))
    for lay in ["a_k/b_k", "a_k/b_mn", "a_mn/b_k", "a_mn/b_mn"]:
        for force in (3, 4):
            try:
                got = T._run(env, a, b, force, transpose_b=lay.endswith("b_k"),
                             a_mn=lay.startswith("a_mn"))
                err = np.abs(got - a @ b).max()
                print(shp, lay, force, f"maxerr {err:.3e}", "ZEROS" if not got.any() else "",
                      flush=True)
            except Exception as e:  # noqa: BLE001
                print(shp, lay, force, "EXC", e, flush=True)
