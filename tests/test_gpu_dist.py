"""GPU, world_size 2 over gloo on one device: both ranks run the B200
Executor on their shard of the iteration space (dist.ShardedPfor, the same
host logic bench.py runs under torchrun/NCCL), and the combined result
matches the unsharded device run.  Sharding changes GEMM shapes (M = the
shard's iterations), so the autotuner may pick other k-splits: results agree
to fp32 rounding (rtol 1e-5), not bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(api, case):
    from paper_1903_04243_b200 import workloads as WL
    if case == "cfg2":
        kw = dict(n=12, model="mlp", d_h=32)
        return 12, ["gather", "sum", "sum", "sum", "sum"], lambda sh: WL.cfg2(api, shard=sh, **kw), \
            lambda: WL.cfg2(api, **kw)
    if case == "cfg3":
        kw = dict(width=64, out_dim=16)
        return 16, ["gather"] * 4, lambda sh: WL.cfg3(api, shard=sh, **kw), lambda: WL.cfg3(api, **kw)
    if case == "cfg4":
        kw = dict(n=6, steps=5, units=16)
        return 6, ["gather", "gather"], lambda sh: WL.cfg4(api, shard=sh, **kw), \
            lambda: WL.cfg4(api, **kw)
    kw = dict(n=9, max_len=7, units=16, masked=True, unroll=2)
    return 9, ["gather"], lambda sh: WL.cfg5(api, shard=sh, **kw), lambda: WL.cfg5(api, **kw)


def _worker(rank, world, port, case, q):
    import torch.distributed as dist
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.dist import ShardedPfor
    from paper_1903_04243_b200.executor import Executor
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        api = WL.this_api()
        n_total, combine, build, full = _case(api, case)
        sp = ShardedPfor(build, n_total, combine, lambda g: Executor(g, device="cuda:0"))
        got = [t.numpy() for t in sp.run()]
        launches = sp.ex.launch_count
        if rank == 0:
            w = full()
            want = [np.asarray(o.data) for o in Executor(w.graph, device="cuda:0").run(feeds=w.feeds)]
            q.put(([g.shape for g in got], [w_.shape for w_ in want],
                   [float(np.max(np.abs(g - w_) / (1e-5 + np.abs(w_)))) if w_.size else 0.0
                    for g, w_ in zip(got, want)], launches))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_two_ranks_b200_executor_match_unsharded(case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    gs, ws, errs, launches = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [tuple(s) for s in gs] == [tuple(s) for s in ws]
    assert launches > 0  # the rank's work ran through the library's kernels
    assert max(errs) < 1e-4, errs
