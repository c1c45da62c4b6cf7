"""GPU: the sm_100a path against the reference's own outputs (golden fixtures)
and the oracle.  Bar: fp32 within rtol 1e-4 / atol 1e-5 of the f64 reference;
integer / index / bool results bit-exact."""

import pathlib

import numpy as np
import pytest

import kernel_graphs as KG
from test_oracle_golden import PROGRAM_CASES, build_program

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5
GOLD = pathlib.Path(__file__).parent / "golden"


@pytest.fixture(scope="module")
def Executor():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1903_04243_b200.executor import Executor
    return Executor


def check(got, want, rtol=RTOL, atol=ATOL):
    want = np.asarray(want)
    assert tuple(got.shape) == tuple(want.shape), (got.shape, want.shape)
    if want.dtype.kind == "f":
        np.testing.assert_allclose(np.asarray(got.data, np.float64), want, rtol=rtol, atol=atol,
                                   equal_nan=True)
    else:
        np.testing.assert_array_equal(np.asarray(got.data).astype(want.dtype), want)


def test_native_library_is_loaded(Executor):
    from paper_1903_04243_b200 import GraphBuilder
    b = GraphBuilder()
    b.graph.set_outputs([b.add(b.f64(np.ones(3)), b.f64(np.ones(3)))])
    (r,) = Executor(b.graph).run()
    np.testing.assert_array_equal(r.data, 2 * np.ones(3))
    maps = pathlib.Path("/proc/self/maps").read_text()
    assert "libpfb.so" in maps


def _kernel_names():
    return [n for n in KG.case_names(np.load(GOLD / "kernels.npz").files) if n != "rng"]


@pytest.mark.parametrize("name", _kernel_names())
def test_kernel_vs_reference(name, golden, Executor):
    K = golden["kernels"]
    g = KG.build_case(name, KG.inputs(K, name))
    ex = Executor(g)
    (got,) = ex.run()
    check(got, K[f"{name}/out"])
    assert ex.launch_count >= 0


def test_rng_vs_reference(golden, Executor):
    from paper_1903_04243_b200 import GraphBuilder
    from paper_1903_04243_b200.executor import RngState
    K = golden["kernels"]
    b = GraphBuilder()
    b.graph.set_outputs([b.random_uniform((4, 5))])
    ex = Executor(b.graph, rng=RngState(int(K["rng/in/seed"]), int(K["rng/in/counter"])))
    (got,) = ex.run()
    np.testing.assert_allclose(got.data, K["rng/out"], rtol=1e-7, atol=0)


@pytest.mark.parametrize("name", sorted(PROGRAM_CASES))
def test_program_vs_reference(name, golden, Executor):
    P = golden["programs"]
    w = build_program(name)
    ex = Executor(w.graph)
    outs = ex.run(feeds=w.feeds)
    for j, o in enumerate(outs):
        check(o, P[f"{name}/out/{j}"])


@pytest.mark.parametrize("name", sorted(PROGRAM_CASES))
def test_program_reference_registry_vs_reference(name, golden, Executor):
    """The unmodified reference formulation (incl. its fallback loops) on device."""
    from paper_1903_04243_b200 import reference_registry
    if PROGRAM_CASES[name][0] == "cfg3":
        pytest.skip("cfg3 takes no registry")
    P = golden["programs"]
    w = build_program(name, registry=reference_registry())
    outs = Executor(w.graph).run(feeds=w.feeds)
    for j, o in enumerate(outs):
        check(o, P[f"{name}/out/{j}"])


@pytest.mark.parametrize("name", ["pairwise_sum_diff", "gather_identity", "matmul_fold",
                                  "conv2d_fold", "reduce_sum_renumber", "concat_shift",
                                  "broadcast_reshape", "cond_example", "while_example"])
def test_worked_example_parfor_graph(name, golden, Executor):
    import worked_examples_local as WE
    g = getattr(WE, name)()  # parfor block: the executor vectorizes it first
    P = golden["programs"]
    for j, o in enumerate(Executor(g).run()):
        check(o, P[f"we_{name}/out/{j}"])


def test_gather_out_of_bounds_raises(Executor):
    from paper_1903_04243_b200 import GraphBuilder, errors
    b = GraphBuilder()
    b.graph.set_outputs([b.gather(b.const(np.ones((4, 3))), b.const(np.array([0, 4])))])
    with pytest.raises(errors.ExecError) as e:
        Executor(b.graph).run()
    assert isinstance(e.value.cause, errors.IndexOutOfBounds)


@pytest.mark.parametrize("idx", [[0, 5, 1], [1, 2, 3, 4]])
def test_gather_out_of_bounds_raises_kernel_and_view(idx, Executor):
    """[0,5,1] goes through the gather kernel (device error word), the
    arithmetic progression through the view path (host check)."""
    from paper_1903_04243_b200 import GraphBuilder, errors
    b = GraphBuilder()
    b.graph.set_outputs([b.gather(b.const(np.ones((4, 3))), b.const(np.array(idx)))])
    with pytest.raises(errors.ExecError) as e:
        Executor(b.graph).run()
    assert isinstance(e.value.cause, errors.IndexOutOfBounds)


@pytest.mark.parametrize("idx", [[2], [0, 1, 2], [1, 3, 5], [4, 4, 4], [5, 3, 0]])
def test_gather_constant_index_values(idx, Executor):
    """Constant progressions become strided views; values as the reference."""
    from paper_1903_04243_b200 import GraphBuilder
    x = np.arange(6 * 5, dtype=np.float64).reshape(6, 5)
    b = GraphBuilder()
    xc = b.const(x)
    g1 = b.gather(xc, b.const(np.array(idx)))
    b.graph.set_outputs([g1, b.mul(g1, b.f64(2.0))])
    got, got2 = Executor(b.graph).run()
    check(got, x[idx])
    check(got2, 2 * x[idx])


@pytest.mark.parametrize("sets,err", [(([0, 1], [1, 2]), "IndexCollision"),
                                      (([0], [2]), "IncompleteCover")])
def test_scatter_rows_validation(sets, err, Executor):
    from paper_1903_04243_b200 import GraphBuilder, errors
    b = GraphBuilder()
    i0, i1 = (b.const(np.array(s, dtype=np.int64)) for s in sets)
    p0 = b.const(np.ones((len(sets[0]), 2)))
    p1 = b.const(np.ones((len(sets[1]), 2)))
    b.graph.set_outputs([b.scatter_rows([i0, i1], [p0, p1], b.i64(3))])
    with pytest.raises(errors.ExecError) as e:
        Executor(b.graph).run()
    assert type(e.value.cause).__name__ == err


def test_dispatch_count_independent_of_output_size(Executor):
    from paper_1903_04243_b200 import GraphBuilder, jacobian
    counts = []
    for m in (4, 32):
        r = np.random.default_rng(m)
        b = GraphBuilder()
        x = b.const(r.standard_normal((8,)))
        W = b.const(r.standard_normal((8, m)))
        y = b.tanh(b.reshape(b.matmul(b.reshape(x, [1, 8]), W), [m]))
        b.graph.set_outputs([jacobian(b, y, x)])
        ex = Executor(b.graph)
        ex.run()
        counts.append(ex.dispatch_count)
    assert counts[0] == counts[1]


@pytest.mark.parametrize("seed", range(6))
def test_random_strided_broadcast_binary(seed, Executor):
    """Transposed / stride-0 views through the elementwise and reduce kernels."""
    from paper_1903_04243_b200 import GraphBuilder
    r = np.random.default_rng(seed)
    a = np.asarray(r.standard_normal((6, 5, 8)), np.float32).astype(np.float64)
    c = np.asarray(r.standard_normal((5, 1)), np.float32).astype(np.float64)
    b = GraphBuilder()
    A = b.transpose(b.const(a), [2, 0, 1])          # [8,6,5] strided view
    T = b.tile_leading(b.const(c[:, 0]), b.i64(6))  # [6,5] stride-0
    s = b.mul(A, T)
    red = b.reduce_sum(s, [seed % 3])
    b.graph.set_outputs([s, red])
    got_s, got_r = Executor(b.graph).run()
    want = np.transpose(a, [2, 0, 1]) * np.broadcast_to(c[:, 0], (6, 5))
    check(got_s, want)
    check(got_r, want.sum(axis=seed % 3))


@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 33, 65), (2, 130, 257), (1, 512, 1024),
                                   (3, 64, 2048)])
def test_matmul_shapes(shape, Executor):
    from paper_1903_04243_b200 import GraphBuilder
    bsz, m, k = shape
    n = (k * 3) // 2 + 1
    r = np.random.default_rng(k)
    a = np.asarray(r.standard_normal((bsz, m, k)), np.float32).astype(np.float64)
    w = np.asarray(r.standard_normal((bsz, k, n)) / np.sqrt(k), np.float32).astype(np.float64)
    b = GraphBuilder()
    b.graph.set_outputs([b.matmul(b.const(a), b.const(w)),
                         b.matmul(b.reshape(b.const(a), [bsz * m, k]), b.const(w[0]))])
    got3, got2 = Executor(b.graph).run()
    check(got3, a @ w)
    check(got2, a.reshape(bsz * m, k) @ w[0])


def test_cuda_graph_replay_tracks_feeds(Executor):
    """Auto CUDA-graph capture: replays must see new feed values and match eager."""
    w = build_program("cfg2_mlp")
    feeds2 = {k: (np.asarray(v) * 0.5 if np.asarray(v).dtype.kind == "f" else v)
              for k, v in w.feeds.items()}
    ex = Executor(w.graph)
    eager = Executor(w.graph, cuda_graph=False)
    want1, want2 = eager.run(w.feeds), eager.run(feeds2)
    got = [ex.run(w.feeds), ex.run(feeds2), ex.run(w.feeds), ex.run(feeds2)]
    assert ex._captures, "pure block-free graph should have been captured"
    for g, want in zip(got, [want1, want2, want1, want2]):
        for a, b in zip(g, want):
            np.testing.assert_allclose(a.data, b.data, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("name", ["cfg2_mlp", "cfg2_conv", "cfg4_mid", "cfg1_full"])
def test_program_unoptimized_vs_reference(name, golden, Executor):
    """The executor with its fusion passes off (one kernel per reference op)."""
    P = golden["programs"]
    w = build_program(name)
    outs = Executor(w.graph, optimize=False, cuda_graph=False).run(feeds=w.feeds)
    for j, o in enumerate(outs):
        check(o, P[f"{name}/out/{j}"])


def test_fusion_reduces_launches(Executor):
    w = build_program("cfg4_mid")
    fused, plain = Executor(w.graph, cuda_graph=False), Executor(w.graph, optimize=False,
                                                                  cuda_graph=False)
    fused.run(feeds=w.feeds)
    plain.run(feeds=w.feeds)
    assert fused.launch_count < 0.7 * plain.launch_count, (fused.launch_count, plain.launch_count)


@pytest.mark.parametrize("unroll", [1, 4])
@pytest.mark.parametrize("name", ["cfg5", "cfg5_mid"])
def test_masked_control_flow_vs_reference(name, unroll, golden, Executor):
    """Predicated while/cond (fixed shapes) on device: reference values; run 1
    is host-driven (its body captured and replayed per trip from trip 2), runs
    2+ execute the whole loop as one CUDA graph with a conditional WHILE node."""
    from paper_1903_04243_b200 import workloads as WL
    _, kw = PROGRAM_CASES[name]
    w = WL.cfg5(WL.this_api(), masked=True, unroll=unroll, **kw)
    ex = Executor(w.graph)
    counts = []
    for _ in range(4):
        c0 = ex.launch_count
        outs = ex.run(feeds=w.feeds)
        counts.append(ex.launch_count - c0)
        for j, o in enumerate(outs):
            check(o, golden["programs"][f"{name}/out/{j}"])
    assert ex._sub_captures, f"loop body not captured: {ex.capture_failures}"
    assert ex._loops, f"device loop not built: {ex.capture_failures}"
    # the device loop's launch accounting matches the host-driven run's
    assert counts[2] == counts[3] and counts[2] > 0, counts


def test_device_loop_host_loop_agree(Executor):
    """Same program with device loops disabled (host-driven trips): identical
    results, bit for bit (same kernels, same order)."""
    from paper_1903_04243_b200 import executor as X
    from paper_1903_04243_b200 import workloads as WL
    w = WL.cfg5(WL.this_api(), masked=True, unroll=2, n=64, max_len=20, units=32)
    ex = Executor(w.graph)
    for _ in range(3):
        dev = ex.run(feeds=w.feeds)
    assert ex._loops, ex.capture_failures
    saved = X._DEVICE_LOOPS
    try:
        X._DEVICE_LOOPS = False
        host = Executor(w.graph).run(feeds=w.feeds)
    finally:
        X._DEVICE_LOOPS = saved
    for a, b in zip(dev, host):
        np.testing.assert_array_equal(np.asarray(a.data), np.asarray(b.data))


def test_replayed_results_stay_valid(Executor):
    """run() of a captured graph returns zero-copy views of pooled pinned
    buffers: results the caller still holds must never be overwritten by
    later runs (pool exhaustion falls back to copies), released buffers are
    reused, and errors words still travel with the packed results."""
    import gc
    w = build_program("cfg2_mlp")
    feeds = [{k: (np.asarray(v) * (0.25 * (i + 1)) if np.asarray(v).dtype.kind == "f" else v)
              for k, v in w.feeds.items()} for i in range(3)]
    eager = Executor(w.graph, cuda_graph=False)
    want = [eager.run(f) for f in feeds]
    ex = Executor(w.graph)
    held = [ex.run(feeds[i % 3]) for i in range(10)]
    assert ex._captures
    for i, res in enumerate(held):
        for a, b in zip(res, want[i % 3]):
            np.testing.assert_allclose(a.data, b.data, rtol=1e-6, atol=1e-7)
    cap = next(iter(ex._captures.values()))
    n_slots = len(cap.host_pack["slots"])
    assert n_slots <= ex._IO_SLOTS + 1
    del held, res, a, b
    gc.collect()
    for i in range(6):
        res = ex.run(feeds[i % 3])
        for a, b in zip(res, want[i % 3]):
            np.testing.assert_allclose(a.data, b.data, rtol=1e-6, atol=1e-7)
    assert len(cap.host_pack["slots"]) == n_slots <= ex._IO_SLOTS + 1


def test_replayed_graph_errors_raise_once(Executor):
    """Device error words of a captured graph travel with its packed results:
    an out-of-range index fed to a replay raises ExecError(IndexOutOfBounds);
    the next valid run does not see stale bits."""
    from paper_1903_04243_b200 import GraphBuilder, errors
    from paper_1903_04243_b200.tensor import DType
    b = GraphBuilder()
    idx = b.placeholder("idx", DType.I64, (3,))
    b.graph.set_outputs([b.gather(b.const(np.arange(12.0).reshape(4, 3)), idx)])
    ex = Executor(b.graph)
    good, bad = {"idx": np.array([0, 3, 1])}, {"idx": np.array([0, 7, 1])}
    for _ in range(3):
        np.testing.assert_allclose(ex.run(good)[0].data, np.arange(12.0).reshape(4, 3)[[0, 3, 1]])
    assert ex._captures
    with pytest.raises(errors.ExecError) as e:
        ex.run(bad)
    assert isinstance(e.value.cause, errors.IndexOutOfBounds)
    np.testing.assert_allclose(ex.run(good)[0].data, np.arange(12.0).reshape(4, 3)[[0, 3, 1]])


@pytest.mark.parametrize("n_in", [8, 70, 200])
def test_concat_many_thin_inputs(n_in, Executor):
    """concat of many width-1 columns along the last axis (cfg4's F2 operand
    path: tiled transpose kernel), inputs as transposed views."""
    from paper_1903_04243_b200 import GraphBuilder
    r = np.random.default_rng(n_in)
    cols = [r.standard_normal((3, 1, 37)) for _ in range(n_in)]
    b = GraphBuilder()
    parts = [b.transpose(b.const(c), [0, 2, 1]) for c in cols]  # [3, 37, 1] views
    b.graph.set_outputs([b.concat(parts, 2)])
    got = Executor(b.graph, cuda_graph=False).run()[0].data
    want = np.concatenate([np.transpose(c, (0, 2, 1)) for c in cols], axis=2)
    np.testing.assert_allclose(np.asarray(got, np.float64), want, rtol=1e-6, atol=1e-7)


_PFG = pathlib.Path(__file__).parent / "golden" / "pfg"


@pytest.mark.parametrize("name", sorted(p.name for p in _PFG.glob("vec_*.pfg")))
def test_reference_pfg_graph_on_device(name, golden, Executor):
    """The reference's own vectorized graphs (its `.pfg` text, loaded by
    paper_1903_04243_b200.pfg) execute on the B200 to the reference outputs."""
    from paper_1903_04243_b200 import pfg
    P = golden["programs"]
    got = Executor(pfg.load(_PFG / name)).run()
    case = "we_" + name[4:-4]
    for j, o in enumerate(got):
        check(o, P[f"{case}/out/{j}"])


@pytest.mark.parametrize("fname,case", [("prog_cfg1_full.pfg", "cfg1_full"),
                                        ("prog_cfg2_mlp.pfg", "cfg2_mlp"),
                                        ("prog_cfg5.pfg", "cfg5")])
def test_reference_pfg_program_on_device(fname, case, golden, Executor):
    from paper_1903_04243_b200 import pfg
    P = golden["programs"]
    feeds = {k.split("/")[-1]: P[k] for k in P if k.startswith(f"{case}/feed/")}
    got = Executor(pfg.load(_PFG / fname)).run(feeds=feeds)
    for j, o in enumerate(got):
        check(o, P[f"{case}/out/{j}"])


def test_reference_random_corpus_on_device(Executor):
    """The reference's 400-case randomized corpus (randgen.py, criterion 1 of
    its acceptance tests), its own vectorized graphs loaded from `.pfg`,
    executed on the B200 (variables, random draws, nested cond/while):
    outputs and final variables against the reference's (random-draw
    dependent ones by shape/dtype, as the reference compares them)."""
    import gzip
    import json
    from paper_1903_04243_b200 import pfg
    from paper_1903_04243_b200.executor import RngState, VariableStore
    corpus = json.load(gzip.open(GOLD / "corpus.json.gz", "rt"))

    def cmp(got, want, tainted):
        if tuple(got.shape) != tuple(want["shape"]) or got.dtype.value != want["dtype"]:
            return f"{got.dtype.value}{list(got.shape)} vs {want['dtype']}{want['shape']}"
        if tainted or not got.data.size:
            return None
        g = np.asarray(got.data, np.float64)
        w = np.asarray(want["data"], np.float64).reshape(want["shape"])
        if want["dtype"] == "f64":
            ok = np.allclose(g, w, rtol=RTOL, atol=ATOL, equal_nan=True)
        else:
            ok = np.array_equal(g, w)
        return None if ok else f"max abs delta {np.max(np.abs(g - w)):.3e}"
    bad = []
    for key, c in corpus.items():
        g = pfg.loads(c["vec"])
        ex = Executor(g, store=VariableStore(g.variables), rng=RngState(c["seed"]))
        try:
            outs = ex.run()
        except Exception as e:  # noqa: BLE001
            bad.append(f"{key}: {type(e).__name__}: {e}")
            continue
        for j, (o, w) in enumerate(zip(outs, c["outs"])):
            msg = cmp(o, w, c["tainted"][j])
            if msg:
                bad.append(f"{key} out {j}: {msg}")
        for name, w in c["vars"].items():
            msg = cmp(ex.store.values[name], w, c["var_tainted"].get(name, False))
            if msg:
                bad.append(f"{key} var {name}: {msg}")
    assert not bad, f"{len(bad)} mismatches: {bad[:8]}"


@pytest.mark.parametrize("d,dt", [(512, "f32"), (6, "f32"), (8, "i64")])
def test_concat_row_strided_slices(d, dt, Executor):
    """concat([x[:, t, :], h], axis=1) with x[:, t, :] a row-strided slice of
    [n, T, d] (cfg4's per-step GEMM operand): the row-copy path reads the
    slice in place (vector and scalar variants), exact."""
    import torch
    from paper_1903_04243_b200 import _native as N
    from paper_1903_04243_b200.executor import DArray
    from paper_1903_04243_b200.tensor import DType
    dev = torch.device("cuda")
    n, T = 37, 5
    tdt, DT = (torch.float32, DType.F64) if dt == "f32" else (torch.int64, DType.I64)
    x = (torch.randn(n, T, d, device=dev) * 100).to(tdt)
    h = (torch.randn(n, d + 4, device=dev) * 100).to(tdt)
    out = torch.empty(n, 2 * d + 4, dtype=tdt, device=dev)
    lib = N.lib()
    for t in (0, 3):
        X = DArray(x.reshape(-1), t * d, (n, d), (T * d, 1), DT)
        H = DArray(h.reshape(-1), 0, tuple(h.shape), h.stride(), DT)
        O = DArray(out.reshape(-1), 0, tuple(out.shape), out.stride(), DT)
        descs = (N.PfbTensor * 2)(X.desc(), H.desc())
        od = O.desc()
        rc = lib.pfb_concat(2, descs, 1, od, torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        want = torch.cat([x[:, t, :], h], dim=1)
        assert torch.equal(out, want)


@pytest.mark.parametrize("shape", [(5, 7, 64), (3, 1000, 12), (2, 333, 128), (4, 3, 4),
                                   (257, 8, 100)])
def test_reduce_short_inner_rows(shape, Executor):
    """inner reductions over short contiguous rows (the several-rows-per-warp
    kernel; cfg4's bias gradient sums T = 64 per row), plus an offset view
    whose rows are not 16-byte aligned (the general warp kernel)."""
    from paper_1903_04243_b200 import GraphBuilder
    r = np.random.default_rng(sum(shape))
    a = np.asarray(r.standard_normal(shape), np.float32).astype(np.float64)
    b = GraphBuilder()
    x = b.const(a)
    red = b.reduce_sum(x, [2])
    tail = b.reduce_sum(b.gather(b.transpose(x, [2, 0, 1]),
                                 b.const(np.arange(1, shape[2], dtype=np.int64))), [0])
    b.graph.set_outputs([red, tail])
    got, got_t = Executor(b.graph).run()
    check(got, a.sum(axis=2))
    check(got_t, np.transpose(a, [2, 0, 1])[1:].sum(axis=0))


@pytest.mark.parametrize("units", [4, 64])
def test_packed_concat_slots_cfg4(units, Executor):
    """F13: cfg4 with packed fused outputs (the forward cell writes the next
    GEMM operand [x_{t+1}, h_t], the backward cell writes dz in place) against
    the oracle on the unoptimized graph."""
    from oracle import OracleExecutor
    from paper_1903_04243_b200 import workloads as WL
    w = WL.cfg4(WL.this_api(), n=8, steps=6, units=units)
    ex = Executor(w.graph)
    got = ex.run(feeds=w.feeds)
    want = OracleExecutor(w.graph).run(feeds=w.feeds)
    for g_, r_ in zip(got, want):
        check(g_, r_.data)
    assert "fused_pack" in {n.kind for n in ex._exec_graph.nodes.values()}


@pytest.mark.parametrize("n_in", [8, 64])
def test_concat_thin_two_level_rows(n_in, Executor):
    """thin concat whose pieces are transposed slices of packed buffers
    ([n, 1, 8w] -> slot [n, 1, 2w] -> [n, 2w, 1]): rows with an outer and an
    inner stride (cfg4's F2 operand after F13)."""
    from paper_1903_04243_b200 import GraphBuilder
    r = np.random.default_rng(n_in)
    w = 24
    bufs = [r.standard_normal((5, 1, 8 * w)) for _ in range(n_in)]
    b = GraphBuilder()
    parts = []
    for bf in bufs:
        v = b.reshape(b.const(bf), [5, 8, w])
        sl = b.gather(b.transpose(v, [1, 0, 2]), b.const(np.array([3, 4], dtype=np.int64)))
        sl = b.reshape(b.transpose(sl, [1, 0, 2]), [5, 1, 2 * w])  # may materialise
        parts.append(b.transpose(sl, [0, 2, 1]))
    b.graph.set_outputs([b.concat(parts, 2)])
    got = Executor(b.graph, cuda_graph=False).run()[0].data
    want = np.concatenate([np.transpose(bf.reshape(5, 8, w)[:, 3:5].reshape(5, 1, 2 * w), (0, 2, 1))
                           for bf in bufs], axis=2)
    np.testing.assert_allclose(np.asarray(got, np.float64), want, rtol=1e-6, atol=1e-7)
