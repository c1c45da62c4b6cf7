"""Intra-GPU sharding experiment: the cfg4 step as K independent example
shards (pfor(shard=...)), each its own Executor / captured CUDA graph replayed
on its own stream, so one shard's latency-bound cell kernels overlap another
shard's GEMMs.  Device time of `steps` steps (all shards), vs one executor.

    python tools/experiments/two_streams.py [--shards 2] [--steps 10]
"""
import argparse
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent.parent))
from paper_1903_04243_b200 import workloads as WL  # noqa: E402
from paper_1903_04243_b200.executor import Executor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--n", type=int, default=256)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    n, K = args.n, args.shards
    full = WL.cfg4(WL.this_api(), n=n)
    feeds = {k: torch.as_tensor(v.astype(np.float32)).to(dev) for k, v in full.feeds.items()}
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    ex = Executor(full.graph, device=dev)
    for _ in range(3):
        ex.run_device(feeds)
    torch.cuda.synchronize()
    st.record()
    for _ in range(args.steps):
        ex.run_device(feeds)
    en.record()
    torch.cuda.synchronize()
    t_one = st.elapsed_time(en) / args.steps
    print(f"one executor: {t_one:.3f} ms/step", flush=True)
    ref = [o.torch_view().clone() for o in ex.run_device(feeds)]
    torch.cuda.synchronize()
    del ex

    per = n // K
    streams = [torch.cuda.Stream(dev) for _ in range(K)]
    exs = []
    for k in range(K):
        w = WL.cfg4(WL.this_api(), n=n, shard=(k * per, (k + 1) * per))
        with torch.cuda.stream(streams[k]):
            e = Executor(w.graph, device=dev)
            for _ in range(3):
                e.run_device(feeds)
        exs.append(e)
    torch.cuda.synchronize()
    main_s = torch.cuda.current_stream(dev)

    def step():
        ev = torch.cuda.Event()
        ev.record(main_s)
        outs = []
        for k in range(K):
            streams[k].wait_event(ev)
            with torch.cuda.stream(streams[k]):
                outs.append(exs[k].run_device(feeds))
        for k in range(K):
            main_s.wait_stream(streams[k])
        return outs

    step()
    torch.cuda.synchronize()
    st.record()
    for _ in range(args.steps):
        step()
    en.record()
    torch.cuda.synchronize()
    t_k = st.elapsed_time(en) / args.steps
    print(f"{K} shards on {K} streams: {t_k:.3f} ms/step ({t_one / t_k:.2f}x)", flush=True)
    outs = step()
    torch.cuda.synchronize()
    err = 0.0
    for j, r in enumerate(ref):
        got = torch.cat([outs[k][j].torch_view() for k in range(K)], 0)
        err = max(err, (got - r).abs().max().item())
    print(f"max |sharded - one| = {err:.2e}")


if __name__ == "__main__":
    main()
