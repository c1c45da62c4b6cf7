"""Where the end-to-end time of Executor.run goes (host side), one config.

    python tools/e2e_profile.py --config cfg2_mlp
"""
import argparse
import cProfile
import pathlib
import pstats
import sys
import time

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1903_04243_b200 import workloads as WL  # noqa: E402
from paper_1903_04243_b200.executor import Executor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2_mlp")
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--raw", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda")
    builder, kw, _ = bench.CONFIGS[args.config]
    w = WL.BUILDERS[builder](WL.this_api(), **kw)
    ex = Executor(w.graph, device=dev, check_errors=False)
    pinned = {k: torch.as_tensor(np.asarray(v, np.float32 if np.asarray(v).dtype == np.float64
                                            else np.asarray(v).dtype)).pin_memory()
              for k, v in w.feeds.items()}
    dfeeds = {k: v.to(dev) for k, v in pinned.items()}
    for _ in range(5):
        ex.run(pinned)
    torch.cuda.synchronize()

    def timeit(fn, n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e6

    print(f"run(pinned host feeds):      {timeit(lambda: ex.run(pinned), args.n):8.1f} us")
    print(f"run_device(device feeds)+sync: {timeit(lambda: (ex.run_device(dfeeds), torch.cuda.synchronize()), args.n):8.1f} us")
    print(f"run_device(pinned feeds)+sync: {timeit(lambda: (ex.run_device(pinned), torch.cuda.synchronize()), args.n):8.1f} us")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(args.n):
        ex.run(pinned)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__" and "--raw" not in sys.argv:
    main()


def raw_floor(config="cfg2_mlp", n=300):
    """run() against the bare replays it performs (Python overhead = the gap)."""
    dev = torch.device("cuda")
    builder, kw, _ = bench.CONFIGS[config]
    w = WL.BUILDERS[builder](WL.this_api(), **kw)
    ex = Executor(w.graph, device=dev, check_errors=False)
    pinned = {k: torch.as_tensor(np.asarray(v, np.float32 if np.asarray(v).dtype == np.float64
                                            else np.asarray(v).dtype)).pin_memory()
              for k, v in w.feeds.items()}
    for _ in range(5):
        res = ex.run(pinned)
    cap = next(iter(ex._captures.values()))
    sl = cap.host_pack["slots"][1]
    static = list(cap.inputs.values())
    src = list(pinned.values())

    def bare():
        for d, s in zip(static, src):
            d.torch_view().copy_(s.reshape(d.torch_view().shape), non_blocking=True)
        cap.graph.replay()
        sl["graph"].replay()
        torch.cuda.current_stream().synchronize()

    def t(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e6
    del res
    print(f"{config}: run() {t(lambda: ex.run(pinned)):.1f} us   bare replays {t(bare):.1f} us")


if __name__ == "__main__" and "--raw" in sys.argv:
    raw_floor()
