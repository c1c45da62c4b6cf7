"""GPU: the tcgen05 3xTF32 GEMM and the SIMT GEMM against f64 numpy, directly
through the C ABI (pfb_matmul_ex, forced path)."""

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


def _run(env, a, b, force, transpose_b=False, accumulate_into=None, alpha=None):
    torch, lib, DArray, DType = env
    dev = torch.device("cuda")
    A = DArray.from_numpy(a, DType.F64, dev)
    if transpose_b:  # K-major B: store B^T densely, pass a transposed view
        Bt = DArray.from_numpy(np.swapaxes(b, -1, -2).copy(), DType.F64, dev)
        perm = list(range(b.ndim))
        perm[-1], perm[-2] = perm[-2], perm[-1]
        B = Bt.view([Bt.shape[p] for p in perm], [Bt.strides[p] for p in perm])
    else:
        B = DArray.from_numpy(b, DType.F64, dev)
    shape = a.shape[:-1] + (b.shape[-1],)
    C = (DArray.from_numpy(accumulate_into, DType.F64, dev) if accumulate_into is not None
         else DArray.empty(shape, DType.F64, dev))
    al = None
    if alpha is not None:
        al_t = torch.as_tensor(alpha.astype(np.float32), device=dev)
        al = al_t.data_ptr()
    ad, bd, cd = A.desc(), B.desc(), C.desc()
    need = lib.pfb_matmul_workspace(ad, bd, cd)
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    rc = lib.pfb_matmul_ex(ad, bd, cd, al, int(accumulate_into is not None), force,
                           ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc
    torch.cuda.synchronize()
    return C.to_numpy().astype(np.float64)


def _f32(r, shape, scale=1.0):
    return np.asarray(r.standard_normal(shape) * scale, np.float32).astype(np.float64)


def _operands(r, a_shape, b_shape):
    """Layer-like scaling (weights ~ 1/sqrt(fan_in)), as in every workload:
    outputs are O(1).  Unscaled N(0,1) operands make even exact-fp32 GEMMs miss
    atol=1e-5 on near-zero outputs once K is in the hundreds."""
    k = a_shape[-1]
    return _f32(r, a_shape), _f32(r, b_shape, 1.0 / np.sqrt(k))


@pytest.mark.parametrize("shape", [(128, 128, 32), (256, 384, 256), (200, 300, 100),
                                   (10240, 784, 256), (513, 129, 1000), (64, 64, 64)])
@pytest.mark.parametrize("force", [1, 2])
def test_gemm_2d(env, shape, force):
    m, n, k = shape
    r = np.random.default_rng(m + n + k)
    a, b = _operands(r, (m, k), (k, n))
    got = _run(env, a, b, force, transpose_b=True)
    np.testing.assert_allclose(got, a @ b, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("force", [1, 2])
def test_gemm_batched(env, force):
    r = np.random.default_rng(7)
    a, b = _operands(r, (3, 160, 96), (3, 96, 200))
    got = _run(env, a, b, force, transpose_b=True)
    np.testing.assert_allclose(got, a @ b, rtol=RTOL, atol=ATOL)


def test_gemm_epilogue_alpha_accumulate(env):
    r = np.random.default_rng(3)
    a, b = _operands(r, (256, 128), (128, 256))
    c0 = _f32(r, (256, 256))
    alpha = np.asarray(r.standard_normal(256), np.float32).astype(np.float64)
    for force in (1, 2):
        got = _run(env, a, b, force, transpose_b=True, accumulate_into=c0, alpha=alpha)
        np.testing.assert_allclose(got, c0 + alpha[:, None] * (a @ b), rtol=RTOL, atol=ATOL)


def test_gemm_tcgen05_is_fp32_accurate_not_tf32(env):
    """Single-pass TF32 would miss by ~1e-3 relative; 3xTF32 must not."""
    r = np.random.default_rng(11)
    a, b = _f32(r, (256, 1024)), _f32(r, (1024, 256))
    got = _run(env, a, b, 2, transpose_b=True)
    want = a @ b
    # error relative to the magnitude scale sqrt(K) of the dot products
    rel = np.max(np.abs(got - want)) / np.sqrt(1024)
    assert rel < 6e-6, rel   # single-pass TF32 gives ~1e-3 here


@pytest.mark.parametrize("k", [64, 1024, 4096])
def test_gemm_tcgen05_matches_simt_error_scale(env, k):
    """3xTF32 error stays within a small factor of the exact-fp32 SIMT error."""
    r = np.random.default_rng(k)
    a, b = _operands(r, (256, k), (k, 256))
    want = a @ b
    e_tc = np.max(np.abs(_run(env, a, b, 2, transpose_b=True) - want))
    e_simt = np.max(np.abs(_run(env, a, b, 1, transpose_b=True) - want))
    assert e_tc < 8 * e_simt + 1e-7, (e_tc, e_simt)


def test_gemm_tcgen05_no_accumulation_bias(env):
    """Truncating in-TMEM accumulation would bias results toward zero linearly
    in K; the chunked RN accumulation must not."""
    r = np.random.default_rng(5)
    a, b = _operands(r, (256, 8192), (8192, 256))
    want = a @ b
    got = _run(env, a, b, 2, transpose_b=True)
    bias = np.mean((got - want) * np.sign(want))
    assert abs(bias) < 5e-7, bias


@pytest.mark.parametrize("shape", [(4096, 1, 4096, 1), (300, 1, 1024, 3), (64, 2, 520, 1)])
def test_small_k_outer_products(env, shape):
    """K<=16 writer paths (cfg3 weight jacobians): exact fp32 products."""
    m, k, n, bsz = shape
    r = np.random.default_rng(m + n)
    a = _f32(r, (bsz, m, k) if bsz > 1 else (m, k))
    b = _f32(r, (bsz, k, n) if bsz > 1 else (k, n))
    got = _run(env, a, b, 0)
    np.testing.assert_allclose(got, a @ b, rtol=1e-6, atol=1e-6)
