"""CPU, world_size 2 over gloo: the sharded pfor (dist.py) reproduces the
unsharded program.  The per-rank compute is the oracle executor (the GPU path
runs the same host logic with the B200 Executor and NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1903_04243_b200.dist import balanced_order, shard_range


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 128, 1000):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_balanced_order_is_a_permutation():
    lengths = np.random.default_rng(0).integers(1, 101, 37)
    perm, inv = balanced_order(lengths, 4)
    assert sorted(perm.tolist()) == list(range(37))
    assert (perm[inv] == np.arange(37)).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    from oracle import OracleExecutor
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.dist import ShardedPfor
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        api = WL.this_api()
        if case == "cfg1_full":
            kw = dict(batch=3, d_in=6, d_h=5, d_out=2, variant="full")
            n_total, combine = 3 * 2, ["gather"]
            build = lambda sh: WL.cfg1(api, shard=sh, **kw)  # noqa: E731
        elif case == "cfg2":
            kw = dict(n=5, model="mlp", d_h=8, materialize=True)
            n_total, combine = 5, ["gather", "sum", "sum", "sum", "sum",
                                   "gather", "gather", "gather", "gather"]
            build = lambda sh: WL.cfg2(api, shard=sh, **kw)  # noqa: E731
        elif case == "cfg5":
            kw = dict(n=7, max_len=5, units=3)
            n_total, combine = 7, ["gather"]
            build = lambda sh: WL.cfg5(api, shard=sh, **kw)  # noqa: E731
        else:
            kw = dict(width=8, out_dim=6)
            n_total, combine = 6, ["gather"] * 4
            build = lambda sh: WL.cfg3(api, shard=sh, **kw)  # noqa: E731
        sp = ShardedPfor(build, n_total, combine, lambda g: OracleExecutor(g))
        got = [t.numpy() for t in sp.run()]
        if rank == 0:
            full = WL.BUILDERS[case.split("_")[0]](api, **kw)
            want = [o.data for o in OracleExecutor(full.graph).run(feeds=full.feeds)]
            if case == "cfg1_full":
                want = [w.reshape(n_total, -1) for w in want]
                got = [g.reshape(n_total, -1) for g in got]
            errs = [float(np.max(np.abs(g - w))) if w.size else 0.0 for g, w in zip(got, want)]
            shapes = [(g.shape, w.shape) for g, w in zip(got, want)]
            q.put((errs, shapes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cfg1_full", "cfg2", "cfg3", "cfg5"])
def test_sharded_pfor_matches_unsharded(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    errs, shapes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for g, w in shapes:
        assert tuple(g) == tuple(w)
    assert max(errs) < 1e-10, errs
