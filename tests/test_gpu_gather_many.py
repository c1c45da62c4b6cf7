"""GPU: pass F17 -- sibling gather_stacked of one operand in one launch
(pfb_gather_stacked_many) against numpy fancy indexing (reference
tensor.gather_rows per iteration, tensor.py:306-318): bit-exact values, and
an out-of-range index of any merged vector raises IndexOutOfBounds naming the
gather it replaced."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1903_04243_b200 import _native as N
    from paper_1903_04243_b200.executor import DArray
    from paper_1903_04243_b200.tensor import DType
    return torch, N, DArray, DType


@pytest.mark.parametrize("n,m,d,q", [(1024, 100, 256, 4), (7, 3, 8, 2), (33, 5, 12, 8)])
def test_gather_many_bit_exact(env, n, m, d, q):
    torch, N, DArray, DType = env
    lib = N.lib()
    dev = torch.device("cuda")
    r = np.random.default_rng(n + q)
    x = r.standard_normal((n, m, d)).astype(np.float32)
    idx = [r.integers(0, m, n).astype(np.int64) for _ in range(q)]
    X = DArray.from_numpy(x, DType.F64, dev)
    I = [DArray.from_numpy(i, DType.I64, dev) for i in idx]
    O = [DArray.empty((n, d), DType.F64, dev) for _ in range(q)]
    err = torch.zeros(q, dtype=torch.int32, device=dev)
    errs = (ctypes.c_void_p * q)(*[err.data_ptr() + 4 * g for g in range(q)])
    rc = lib.pfb_gather_stacked_many(X.desc(), q, (N.PfbTensor * q)(*[i.desc() for i in I]),
                                     (N.PfbTensor * q)(*[o.desc() for o in O]), errs, None)
    assert rc == 0
    torch.cuda.synchronize()
    for g in range(q):
        np.testing.assert_array_equal(O[g].to_numpy(), x[np.arange(n), idx[g]])
    assert not err.any()
    # one out-of-range entry in vector 1 sets that vector's error word only
    bad = idx[1].copy()
    bad[n // 2] = m
    I[1] = DArray.from_numpy(bad, DType.I64, dev)
    rc = lib.pfb_gather_stacked_many(X.desc(), q, (N.PfbTensor * q)(*[i.desc() for i in I]),
                                     (N.PfbTensor * q)(*[o.desc() for o in O]), errs, None)
    assert rc == 0
    torch.cuda.synchronize()
    e = err.cpu().numpy()
    assert e[1] & N.DEV_OOB and not e[0] and not e[2:].any()


def test_gather_many_declines_unaligned_rows(env):
    torch, N, DArray, DType = env
    lib = N.lib()
    dev = torch.device("cuda")
    X = DArray.from_numpy(np.zeros((4, 3, 6), np.float32), DType.F64, dev)
    I = [DArray.from_numpy(np.zeros(4, np.int64), DType.I64, dev) for _ in range(2)]
    O = [DArray.empty((4, 6), DType.F64, dev) for _ in range(2)]
    rc = lib.pfb_gather_stacked_many(X.desc(), 2, (N.PfbTensor * 2)(*[i.desc() for i in I]),
                                     (N.PfbTensor * 2)(*[o.desc() for o in O]), None, None)
    assert rc == N.E_UNSUPPORTED


def test_cfg5_merged_gathers_raise_out_of_range(env):
    """A length past max_len makes the merged per-trip gathers read x[j, t]
    with t = max_len: ExecError(IndexOutOfBounds) from the device loop, as
    with one gather per step."""
    torch, N, DArray, DType = env
    from paper_1903_04243_b200 import errors, workloads as WL
    from paper_1903_04243_b200.executor import Executor
    w = WL.BUILDERS["cfg5"](WL.this_api(), n=64, max_len=8, units=32, masked=True, unroll=4)
    feeds = dict(w.feeds)
    ok = Executor(w.graph, device="cuda:0").run(feeds=feeds)
    assert ok
    lengths = np.array(feeds["lengths"]).copy()
    lengths[5] = 9
    feeds["lengths"] = lengths
    with pytest.raises(errors.ExecError) as e:
        Executor(w.graph, device="cuda:0").run(feeds=feeds)
    assert isinstance(e.value.cause, errors.IndexOutOfBounds)


def test_cfg5_device_loop_trips_and_launches(env):
    """The predicated device loop of cfg5 (unroll 4): one pass of the head and
    exactly ceil(max(lengths) / 4) trips per run (the loop test any(active)
    is set by the write-back kernel, pfb_copy_many_cond), and per trip only
    the per-step work plus the trip's index group, merged gather and
    write-back: 4 GEMMs + 4 select groups + 3 launches."""
    torch, N, DArray, DType = env
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor
    w = WL.BUILDERS["cfg5"](WL.this_api(), n=512, max_len=23, units=256, masked=True, unroll=4)
    ex = Executor(w.graph, device="cuda:0")
    for _ in range(3):
        ex.run(feeds=w.feeds)
    assert ex._loops, ex.capture_failures
    (lp,) = ex._loops.values()
    assert lp.iter_launches <= 11, lp.iter_launches
    c0 = int(lp.counter.item())
    ex.run(feeds=w.feeds)
    torch.cuda.synchronize()
    trips = -(-int(np.max(w.feeds["lengths"])) // 4)
    assert int(lp.counter.item()) - c0 == 1 + trips


def test_replay_reads_device_feeds_in_place(env):
    """run_device with the same device tensors: from the second run on, the
    captured graph reads the feeds in place (no copy into static inputs), and
    it sees in-place updates of them; results equal a fresh executor's."""
    torch, N, DArray, DType = env
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor
    w = WL.BUILDERS["cfg2"](WL.this_api(), n=32, model="mlp")
    dev = torch.device("cuda:0")
    feeds = {k: torch.as_tensor(np.asarray(v, np.float32)).to(dev) for k, v in w.feeds.items()}
    ex = Executor(w.graph, device="cuda:0")
    for _ in range(4):
        ex.run_device(feeds)
    assert any(len(k) == 3 for k in ex._captures), list(ex._captures)
    feeds["x"].mul_(0.5)
    got = [o.to_numpy() for o in ex.run_device(feeds)]
    want = Executor(w.graph, device="cuda:0", cuda_graph=False).run(
        feeds={k: v.cpu().numpy() for k, v in feeds.items()})
    for g_, w_ in zip(got, want):
        np.testing.assert_allclose(np.asarray(g_, np.float64), np.asarray(w_.data, np.float64),
                                   rtol=1e-5, atol=1e-6)
