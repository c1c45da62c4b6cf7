// pfb_matmul: validation + path selection (reference tensor.py:195-206).
#include <algorithm>
#include <cstdlib>

#include "gemm.cuh"

using namespace pfb;

static int matmul_args(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out, GemmArgs* g) {
  if (a->dtype != b->dtype) return PFB_E_DTYPE;
  if (a->dtype != PFB_F32 || out->dtype != PFB_F32) return PFB_E_DTYPE;  // int matmul: not on the path
  if (a->rank == 2 && b->rank == 2) {
    if (a->shape[1] != b->shape[0]) return PFB_E_SHAPE;
    if (out->rank != 2 || out->shape[0] != a->shape[0] || out->shape[1] != b->shape[1])
      return PFB_E_SHAPE;
    *g = GemmArgs{1, a->shape[0], b->shape[1], a->shape[1],
                  (const float*)a->data, 0, a->stride[0], a->stride[1],
                  (const float*)b->data, 0, b->stride[0], b->stride[1],
                  (float*)out->data, 0, out->stride[0], out->stride[1], nullptr, 0};
    return 0;
  }
  if (a->rank == 3 && b->rank == 3) {
    if (a->shape[0] != b->shape[0] || a->shape[2] != b->shape[1]) return PFB_E_SHAPE;
    if (out->rank != 3 || out->shape[0] != a->shape[0] || out->shape[1] != a->shape[1] ||
        out->shape[2] != b->shape[2])
      return PFB_E_SHAPE;
    *g = GemmArgs{a->shape[0], a->shape[1], b->shape[2], a->shape[2],
                  (const float*)a->data, a->stride[0], a->stride[1], a->stride[2],
                  (const float*)b->data, b->stride[0], b->stride[1], b->stride[2],
                  (float*)out->data, out->stride[0], out->stride[1], out->stride[2], nullptr, 0};
    return 0;
  }
  return PFB_E_RANK;
}

__global__ void zero_f32(float* p, int64_t n) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.f;
}

extern "C" int64_t pfb_matmul_workspace(const pfb_tensor* a, const pfb_tensor* b,
                                        pfb_tensor* out) {
  GemmArgs g;
  if (matmul_args(a, b, out, &g)) return 0;
  return std::max(gemm_tcgen05_workspace(g), gemm_simt_workspace(g));
}

extern "C" int pfb_matmul_ex(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                             const float* alpha_rows, int32_t accumulate, int32_t force_path,
                             void* ws, int64_t ws_bytes, void* stream) {
  GemmArgs g;
  if (int e = matmul_args(a, b, out, &g)) return e;
  g.alpha_rows = alpha_rows;
  g.accumulate = accumulate;
  cudaStream_t s = as_stream(stream);
  if (g.batch == 0 || g.M == 0 || g.N == 0) return 0;
  if (g.K == 0) {
    if (accumulate) return 0;
    if (!is_dense(out)) return PFB_E_UNSUPPORTED;
    int64_t n = numel(out);
    launch(zero_f32, grid_for(n, 256), 256, 0, s, (float*)out->data, n);
    return launch_status();
  }
  // force_path: 0 = auto, 1 = SIMT, 2 = tcgen05 (error if ineligible).
  // PFB_DISABLE_TCGEN05=1 pins auto to SIMT (A/B testing, bring-up).
  static const bool tc_off = getenv("PFB_DISABLE_TCGEN05") && getenv("PFB_DISABLE_TCGEN05")[0] == '1';
  if (force_path == 2 || (force_path == 0 && !tc_off && gemm_tcgen05_profitable(g) &&
                          gemm_tcgen05_eligible(g))) {
    int e = gemm_tcgen05(g, ws, ws_bytes, s);
    if (e != PFB_E_UNSUPPORTED || force_path == 2) return e;
  }
  return gemm_simt(g, ws, ws_bytes, s);
}

extern "C" int pfb_matmul(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out, void* ws,
                          int64_t ws_bytes, void* stream) {
  return pfb_matmul_ex(a, b, out, nullptr, 0, 0, ws, ws_bytes, stream);
}
