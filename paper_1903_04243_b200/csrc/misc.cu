// Library info + fused per-example statistics.
#include "common.cuh"

using namespace pfb;

extern "C" int pfb_version(void) { return 100; }

extern "C" int pfb_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

namespace pfb {
// sq_norm[i] += (sum_j a[i,j]^2) * (sum_k b[i,k]^2): one block per example.
__global__ void outer_sq_norm_kernel(int64_t n, int64_t da, int64_t db, const float* a,
                                     int64_t sa0, int64_t sa1, const float* b, int64_t sb0,
                                     int64_t sb1, float* out) {
  pdl_enter();
  __shared__ float red[2][8];
  int64_t i = blockIdx.x;
  float sa = 0.f, sb = 0.f;
  for (int64_t j = threadIdx.x; j < da; j += blockDim.x) {
    float v = a[i * sa0 + j * sa1];
    sa = fmaf(v, v, sa);
  }
  for (int64_t k = threadIdx.x; k < db; k += blockDim.x) {
    float v = b[i * sb0 + k * sb1];
    sb = fmaf(v, v, sb);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = sa;
    red[1][threadIdx.x >> 5] = sb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float ta = 0.f, tb = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { ta += red[0][w]; tb += red[1][w]; }
    out[i] += ta * tb;
  }
}
}  // namespace pfb

extern "C" int pfb_outer_sq_norm(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* sq_norm,
                                 void* stream) {
  if (a->rank != 2 || b->rank != 2 || a->shape[0] != b->shape[0]) return PFB_E_SHAPE;
  if (sq_norm->rank != 1 || sq_norm->shape[0] != a->shape[0] || !is_dense(sq_norm)) return PFB_E_SHAPE;
  int64_t n = a->shape[0];
  if (n == 0) return 0;
  launch(outer_sq_norm_kernel, (unsigned)n, 256, 0, as_stream(stream), 
      n, a->shape[1], b->shape[1], (const float*)a->data, a->stride[0], a->stride[1],
      (const float*)b->data, b->stride[0], b->stride[1], (float*)sq_norm->data);
  return launch_status();
}
