"""Per-launch device time of one step of a bench config, each launch re-issued
alone between CUDA events (warm L2, as inside a step).  The sum against the
graph-replayed step time shows the launch/dependency overhead.

    python tools/launch_breakdown.py --config cfg4 [--top 30]
"""
import argparse
import collections
import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1903_04243_b200 import workloads as WL  # noqa: E402
from paper_1903_04243_b200.executor import Executor  # noqa: E402


def _shapes(fargs):
    """shapes of the tensor descriptors among a launch's C-ABI arguments"""
    out = []
    for a in fargs:
        a = getattr(a, "_obj", a)
        if hasattr(a, "rank") and hasattr(a, "shape"):
            out.append(tuple(a.shape[:a.rank]))
    return " ".join(str(list(x)) for x in out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2_mlp")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda")
    builder, kw, _ = bench.CONFIGS[args.config]
    w = WL.BUILDERS[builder](WL.this_api(), **kw)
    ex = Executor(w.graph, device=dev, check_errors=False)
    feeds = {k: torch.as_tensor(np.asarray(v, np.float32 if np.asarray(v).dtype == np.float64
                                           else np.asarray(v).dtype)).to(dev)
             for k, v in w.feeds.items()}
    for _ in range(4):
        ex.run_device(feeds)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        ex.run_device(feeds)
    e.record()
    torch.cuda.synchronize()
    step_us = s.elapsed_time(e) / 5 * 1e3
    ex.kernel_timer = []
    ex.run_device(feeds)
    torch.cuda.synchronize()
    recs, ex.kernel_timer = ex.kernel_timer, None
    rows = []
    for what, nbytes, flops, _, _, fn, fargs in recs:
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn(*fargs)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        rows.append((float(np.median(ts)), what, nbytes, flops, _shapes(fargs)))
    tot = sum(r[0] for r in rows)
    print(f"{args.config}: step (replayed) {step_us:.1f} us, {len(rows)} launches, "
          f"sum of isolated launches {tot:.1f} us")
    agg = collections.defaultdict(lambda: [0.0, 0, 0, 0])
    for t, what, nb, fl, _ in rows:
        a = agg[what]
        a[0] += t
        a[1] += 1
        a[2] += nb
        a[3] += fl
    for what, (t, n, nb, fl) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"  {what:14s} n={n:5d} {t:10.1f} us {100 * t / tot:5.1f}%  "
              f"{nb / max(t, 1e-9) / 1e3:8.1f} GB/s  {fl / max(t, 1e-9) / 1e6:8.2f} TFLOP/s")
    print("  slowest launches:")
    for t, what, nb, fl, shp in sorted(rows, reverse=True)[:args.top]:
        print(f"    {t:9.2f} us  {what:14s} {nb / 1e6:9.2f} MB  {fl / 1e9:8.3f} GFLOP  {shp}")


if __name__ == "__main__":
    main()
