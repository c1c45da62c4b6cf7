"""GPU: pass F15 -- split-K partials GEMM (pfb_matmul_parts) and fused groups
that sum the partials as they load (pfb_fused_ew_parts), against f64 numpy
(reference tensor.matmul, tensor.py:195-206) and against the executor with
partials disabled."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-5


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1903_04243_b200 import _native as N
    from paper_1903_04243_b200.executor import DArray
    from paper_1903_04243_b200.tensor import DType
    return torch, N.lib(), DArray, DType


def _parts(env, a, b, bias=None, planes=False, b_kmajor=True):
    torch, lib, DArray, DType = env
    dev = torch.device("cuda")
    A = DArray.from_numpy(a, DType.F64, dev)
    if b_kmajor:  # the executor's weights: B^T stored densely ([N, K]), B a transposed view
        Bt = DArray.from_numpy(b.T.copy(), DType.F64, dev)
        B = Bt.view((b.shape[0], b.shape[1]), (1, b.shape[0]))
    else:
        B = DArray.from_numpy(b, DType.F64, dev)
    m, n = a.shape[0], b.shape[1]
    probe = DArray.empty((m, n), DType.F64, dev)
    ad, bd = A.desc(), B.desc()
    S = lib.pfb_matmul_parts_count(ad, bd, probe.desc())
    if S < 1:
        return None, 0
    P = DArray.empty((S, m, n), DType.F64, dev)
    pb = None
    if planes:
        pb = torch.empty(lib.pfb_gemm_planes_bytes(bd), dtype=torch.uint8, device=dev)
        assert lib.pfb_gemm_split_planes(bd, pb.data_ptr(), None) == 0
    need = lib.pfb_matmul_parts_workspace(ad, bd, probe.desc())
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    xd = None
    if bias is not None:
        X = DArray.from_numpy(bias, DType.F64, dev)
        xd = ctypes.byref(X.desc())
    rc = lib.pfb_matmul_parts(ad, bd, P.desc(), xd, pb.data_ptr() if pb is not None else None,
                              ws.data_ptr(), ws.numel(), None)
    assert rc == 0
    torch.cuda.synchronize()
    return P.to_numpy(), S


@pytest.mark.parametrize("m,n,k", [(256, 2048, 1024), (256, 512, 2048), (256, 2048, 512),
                                   (200, 600, 600), (130, 1028, 520)])
@pytest.mark.parametrize("planes", [False, True])
def test_matmul_parts_sum_matches_f64(env, m, n, k, planes):
    r = np.random.default_rng(m + n + k)
    a = r.standard_normal((m, k)).astype(np.float32)
    b = (r.standard_normal((k, n)) / np.sqrt(k)).astype(np.float32)
    bias = r.standard_normal((n,)).astype(np.float32)
    parts, S = _parts(env, a, b, bias, planes)
    assert S >= 1 and parts is not None
    got = parts.astype(np.float64).sum(0)
    want = a.astype(np.float64) @ b.astype(np.float64) + bias
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_matmul_parts_declines_small_products(env):
    """cfg1's 32x256x784 forward GEMM stays on the autotuned reduced paths."""
    torch, lib, DArray, DType = env
    dev = torch.device("cuda")
    a = DArray.empty((32, 784), DType.F64, dev)
    b = DArray.empty((784, 256), DType.F64, dev)
    c = DArray.empty((32, 256), DType.F64, dev)
    assert lib.pfb_matmul_parts_count(a.desc(), b.desc(), c.desc()) == 0
    # and rows of N = 1030 floats (not 16-byte aligned) are declined, not failed
    a2 = DArray.empty((256, 1024), DType.F64, dev)
    b2 = DArray.empty((1024, 1030), DType.F64, dev)
    c2 = DArray.empty((256, 1030), DType.F64, dev)
    assert lib.pfb_matmul_parts_count(a2.desc(), b2.desc(), c2.desc()) == 0


def test_matmul_parts_row_bias_and_row_major_b(env):
    r = np.random.default_rng(7)
    a = r.standard_normal((256, 640)).astype(np.float32)
    b = (r.standard_normal((640, 512)) / 25).astype(np.float32)
    bias = r.standard_normal((256, 512)).astype(np.float32)  # a full matrix addend
    parts, S = _parts(env, a, b, bias, planes=False, b_kmajor=False)
    assert S >= 2
    want = a.astype(np.float64) @ b.astype(np.float64) + bias
    np.testing.assert_allclose(parts.astype(np.float64).sum(0), want, rtol=RTOL, atol=ATOL)


def test_fused_parts_feed_sums_in_split_order(env):
    """An elementwise program over partials: each input summed left to right
    in fp32 as loaded -- bit-identical to numpy's fp32 left fold."""
    torch, lib, DArray, DType = env
    from paper_1903_04243_b200 import _native as N
    dev = torch.device("cuda")
    r = np.random.default_rng(3)
    S, shape = 5, (64, 96)
    parts = r.standard_normal((S,) + shape).astype(np.float32)
    c = r.standard_normal(shape).astype(np.float32)
    P = DArray.from_numpy(parts, DType.F64, dev)
    C = DArray.from_numpy(c, DType.F64, dev)
    view = P.view(shape, P.strides[1:])
    out = DArray.empty(shape, DType.F64, dev)
    # program: r0 = load in0 (partials); r1 = load in1; r3 = tanh(r0) * r1
    ops = _opcodes()
    prog = [(64, 0, 0, 0), (64, 1, 1, 0), (ops["tanh"], 2, 0, 0), (ops["mul"], 3, 2, 1)]
    flat = (ctypes.c_int32 * 16)(*[x for st in prog for x in st])
    spec = (ctypes.c_int64 * 4)(S, int(np.prod(shape)), 1, 0)
    ins = (N.PfbTensor * 2)(view.desc_part0(), C.desc())
    outs = (N.PfbTensor * 1)(out.desc())
    regs = (ctypes.c_int32 * 1)(3)
    if not lib.pfb_fused_parts_ok():
        pytest.skip("specialiser unavailable")
    assert lib.pfb_fused_ew_parts(2, ins, spec, 4, flat, 1, regs, outs, None) == 0
    torch.cuda.synchronize()
    acc = parts[0].copy()
    for j in range(1, S):
        acc = (acc + parts[j]).astype(np.float32)
    got = out.to_numpy()
    want = (np.tanh(acc.astype(np.float64)) * c).astype(np.float32)
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-6)
    # the sum itself is exact in split order: program r2 = r0 (move)
    prog2 = [(64, 0, 0, 0), (64, 1, 1, 0), (ops["add"], 2, 0, 1)]
    flat2 = (ctypes.c_int32 * 12)(*[x for st in prog2 for x in st])
    zero = DArray.from_numpy(np.zeros(shape, np.float32), DType.F64, dev)
    ins2 = (N.PfbTensor * 2)(view.desc_part0(), zero.desc())
    regs2 = (ctypes.c_int32 * 1)(2)
    assert lib.pfb_fused_ew_parts(2, ins2, spec, 3, flat2, 1, regs2, outs, None) == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.to_numpy(), acc)


def _opcodes():
    from paper_1903_04243_b200 import passes
    return {"add": passes._BIN_CODE["add"], "mul": passes._BIN_CODE["mul"],
            "tanh": 16 + passes._UN_CODE["tanh"]}


def test_cfg4_partials_match_reduced_executor(env, monkeypatch):
    """The LSTM program (cfg4 shapes with M = 256 examples, where the per-step
    GEMMs take the partials path) equals the same program with F15 off."""
    torch, lib, DArray, DType = env
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor
    w = WL.BUILDERS["cfg4"](WL.this_api(), n=256, steps=4, units=256)
    ex = Executor(w.graph, device="cuda:0", cuda_graph=False)
    got = ex.run(feeds=w.feeds)
    # every per-step GEMM (4 forward, 3 backward) returned partials and every
    # consumer summed them on load
    assert ex.parts_made == 7 and ex.parts_reduced == 0, (ex.parts_made, ex.parts_reduced)
    ex2 = Executor(w.graph, device="cuda:0")
    monkeypatch.setattr(ex2._lib, "pfb_fused_parts_ok", lambda: 0)
    want = ex2.run(feeds=w.feeds)
    for g_, w_ in zip(got, want):
        np.testing.assert_allclose(np.asarray(g_.data, np.float64), np.asarray(w_.data, np.float64),
                                   rtol=RTOL, atol=ATOL)



@pytest.mark.parametrize("m,n,k1,k2", [(1024, 256, 256, 256), (520, 264, 96, 440)])
def test_matmul_dual_parts_sum_matches_f64(env, m, n, k1, k2):
    """a1 @ b1 + a2 @ b2 (cfg5's RNN cell) as split-K partials over both K ranges."""
    torch, lib, DArray, DType = env
    dev = torch.device("cuda")
    r = np.random.default_rng(m + k1)
    a1 = r.standard_normal((m, k1)).astype(np.float32)
    a2 = r.standard_normal((m, k2)).astype(np.float32)
    b1 = (r.standard_normal((k1, n)) / 16).astype(np.float32)
    b2 = (r.standard_normal((k2, n)) / 16).astype(np.float32)
    A1, A2 = DArray.from_numpy(a1, DType.F64, dev), DArray.from_numpy(a2, DType.F64, dev)
    B1, B2 = DArray.from_numpy(b1, DType.F64, dev), DArray.from_numpy(b2, DType.F64, dev)
    probe = DArray.empty((m, n), DType.F64, dev)
    d = [x.desc() for x in (A1, B1, A2, B2)]
    S = lib.pfb_matmul_dual_parts_count(d[0], d[1], d[2], d[3], probe.desc())
    assert S >= 2
    P = DArray.empty((S, m, n), DType.F64, dev)
    need = lib.pfb_matmul_dual_parts_workspace(d[0], d[1], d[2], d[3], probe.desc())
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    assert lib.pfb_matmul_dual_parts(d[0], d[1], d[2], d[3], P.desc(), None, None, None,
                                     ws.data_ptr(), ws.numel(), None) == 0
    torch.cuda.synchronize()
    want = a1.astype(np.float64) @ b1 + a2.astype(np.float64) @ b2
    np.testing.assert_allclose(P.to_numpy().astype(np.float64).sum(0), want, rtol=RTOL, atol=ATOL)


def test_cfg5_partials_match_reduced_executor(env, monkeypatch):
    """cfg5 (masked, unrolled device loop): the per-trip dual GEMMs return
    partials, summed by the row-sum reduction and the select group."""
    torch, lib, DArray, DType = env
    from paper_1903_04243_b200 import workloads as WL
    from paper_1903_04243_b200.executor import Executor
    w = WL.BUILDERS["cfg5"](WL.this_api(), n=512, max_len=12, units=256, masked=True, unroll=4)
    ex = Executor(w.graph, device="cuda:0", cuda_graph=False)
    got = ex.run(feeds=w.feeds)
    # the row sums read the partials directly (pfb_row_sum_parts) and the
    # select group sums them on load: nothing is reduced into a tensor
    assert ex.parts_made > 0 and ex.parts_reduced == 0, (ex.parts_made, ex.parts_reduced)
    ex2 = Executor(w.graph, device="cuda:0", cuda_graph=False)
    monkeypatch.setattr(ex2._lib, "pfb_fused_parts_ok", lambda: 0)
    want = ex2.run(feeds=w.feeds)
    for g_, w_ in zip(got, want):
        np.testing.assert_allclose(np.asarray(g_.data, np.float64), np.asarray(w_.data, np.float64),
                                   rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("rows,W,S", [(1024, 256, 3), (37, 1024, 1), (300, 64, 2), (5, 40, 1),
                                      (129, 10, 2), (128, 10, 1), (33, 3, 1), (50, 32, 1)])
def test_fused_row_sum_feed(env, rows, W, S):
    """pfb_fused_ew_rows (pass F16): input 1 is the row sum of input 0 (its
    split-K partials summed first), computed inside the group's kernel;
    against f64 numpy.  Rows that are not a whole number of warps are
    declined (PFB_E_UNSUPPORTED) for the executor's materialised fallback;
    rows shorter than a warp share warps (lanes padded to a power of two)."""
    torch, lib, DArray, DType = env
    from paper_1903_04243_b200 import _native as N
    if not lib.pfb_fused_parts_ok():
        pytest.skip("specialiser unavailable")
    dev = torch.device("cuda")
    r = np.random.default_rng(rows + W)
    shape = (rows, 1, W)
    parts = r.standard_normal((S,) + shape).astype(np.float32)
    c = r.standard_normal(shape).astype(np.float32)
    P = DArray.from_numpy(parts, DType.F64, dev)
    C = DArray.from_numpy(c, DType.F64, dev)
    x = P.view(shape, P.strides[1:])
    rs = x.view((rows, 1, 1), (x.strides[0], 0, 0))
    out = DArray.empty(shape, DType.F64, dev)
    ops = _opcodes()
    # r0 = in0 (partials), r1 = in1 (row sum of in0), r2 = in2; r3 = r1 * r2 + r0
    prog = [(64, 0, 0, 0), (64, 1, 1, 0), (64, 2, 2, 0), (ops["mul"], 3, 1, 2),
            (ops["add"], 4, 3, 0)]
    flat = (ctypes.c_int32 * 20)(*[v for st in prog for v in st])
    spec = (ctypes.c_int64 * 6)(S, rows * W, 1, 0, 1, 0)
    rsum = (ctypes.c_int32 * 3)(-1, 0, -1)
    ins = (N.PfbTensor * 3)(x.desc_part0(), rs.desc_part0(), C.desc())
    outs = (N.PfbTensor * 1)(out.desc())
    regs = (ctypes.c_int32 * 1)(4)
    rc = lib.pfb_fused_ew_rows(3, ins, spec, rsum, 5, flat, 1, regs, outs, None)
    if W % 32 and W > 32:
        assert rc == N.E_UNSUPPORTED
        return
    assert rc == 0
    torch.cuda.synchronize()
    z = parts.astype(np.float64).sum(0)
    want = z.sum(axis=2, keepdims=True) * c + z
    np.testing.assert_allclose(out.to_numpy().astype(np.float64), want, rtol=RTOL,
                               atol=ATOL * np.sqrt(W) * 4)


@pytest.mark.parametrize("rows,W", [(128, 10), (300, 256), (7, 1)])
def test_fused_row_sum_of_exp_is_softmax(env, rows, W):
    """pfb_fused_ew_rows with a summand op: rowsum[1] = 0 | (16 + exp) << 16
    makes input 1 the row sum of exp(input 0); the program exp(in0) / in1 is
    the softmax (cfg2's cross-entropy), against f64 numpy."""
    torch, lib, DArray, DType = env
    from paper_1903_04243_b200 import _native as N, passes
    if not lib.pfb_fused_parts_ok():
        pytest.skip("specialiser unavailable")
    dev = torch.device("cuda")
    r = np.random.default_rng(rows * W)
    z = r.standard_normal((rows, 1, W)).astype(np.float32)
    Z = DArray.from_numpy(z, DType.F64, dev)
    rs = Z.view((rows, 1, 1), (Z.strides[0], 0, 0))
    out = DArray.empty((rows, 1, W), DType.F64, dev)
    EXP = 16 + passes._UN_CODE["exp"]
    prog = [(64, 0, 0, 0), (EXP, 0, 0, 0), (64, 1, 1, 0), (passes._BIN_CODE["div"], 2, 0, 1)]
    flat = (ctypes.c_int32 * 16)(*[v for st in prog for v in st])
    rsum = (ctypes.c_int32 * 2)(-1, 0 | (EXP << 16))
    ins = (N.PfbTensor * 2)(Z.desc(), rs.desc())
    outs = (N.PfbTensor * 1)(out.desc())
    regs = (ctypes.c_int32 * 1)(2)
    rc = lib.pfb_fused_ew_rows(2, ins, None, rsum, 4, flat, 1, regs, outs, None)
    if W == 1:  # a one-element row collapses into the outer dims: declined (the
        assert rc == N.E_UNSUPPORTED  # executor then materialises the sums)
        return
    assert rc == 0
    torch.cuda.synchronize()
    e = np.exp(z.astype(np.float64))
    np.testing.assert_allclose(out.to_numpy(), e / e.sum(axis=2, keepdims=True), rtol=1e-5, atol=1e-7)


def test_col_dots_many_operands(env):
    """pfb_col_dots (pass F19): weighted column sums of several operands with
    one weight vector (strided and transposed views included), against f64."""
    torch, lib, DArray, DType = env
    from paper_1903_04243_b200 import _native as N
    dev = torch.device("cuda")
    r = np.random.default_rng(7)
    R = 128
    y = r.standard_normal(R).astype(np.float32)
    xs = [r.standard_normal((R, c)).astype(np.float32) for c in (256, 10, 33)]
    Y = DArray.from_numpy(y.reshape(R, 1), DType.F64, dev)
    X = [DArray.from_numpy(x, DType.F64, dev) for x in xs[:2]]
    xt = DArray.from_numpy(xs[2].T.copy(), DType.F64, dev)  # a transposed view
    X.append(xt.view((R, 33), (1, R)))
    O = [DArray.empty((x.shape[1],), DType.F64, dev) for x in xs]
    assert lib.pfb_col_dots(3, (N.PfbTensor * 3)(*[x.desc() for x in X]), Y.desc(),
                            (N.PfbTensor * 3)(*[o.desc() for o in O]), None) == 0
    torch.cuda.synchronize()
    for x, o in zip(xs, O):
        np.testing.assert_allclose(o.to_numpy(), (x.astype(np.float64) * y[:, None]).sum(0),
                                   rtol=RTOL, atol=ATOL)
