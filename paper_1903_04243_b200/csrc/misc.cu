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

// ---------------------------------------------------------------------------
// pack: several dense tensors -> one byte buffer (one launch), so a run's
// outputs (and its device error words) come back in a single D2H copy.

namespace pfb {
constexpr int kMaxPack = 16;
struct PackDesc {
  const uint8_t* src[kMaxPack];
  int64_t off[kMaxPack];
  int64_t bytes[kMaxPack];
};

__global__ void __launch_bounds__(256) pack_kernel(PackDesc d, uint8_t* dst) {
  pdl_enter();
  const int t = blockIdx.y;
  const uint8_t* s = d.src[t];
  uint8_t* o = dst + d.off[t];
  const int64_t nb = d.bytes[t];
  const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(o)) & 15) == 0;
  const int64_t n16 = vec ? nb / 16 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride)
    reinterpret_cast<int4*>(o)[i] = __ldg(reinterpret_cast<const int4*>(s) + i);
  for (int64_t i = 16 * n16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += stride)
    o[i] = s[i];
}
}  // namespace pfb

extern "C" int pfb_pack(int32_t n, const pfb_tensor* xs, void* dst, const int64_t* dst_offsets,
                        void* stream) {
  if (n < 0) return PFB_E_ARG;
  cudaStream_t s = as_stream(stream);
  for (int base = 0; base < n; base += kMaxPack) {
    PackDesc d = {};
    const int m = n - base < kMaxPack ? n - base : kMaxPack;
    int64_t most = 0;
    for (int j = 0; j < m; ++j) {
      const pfb_tensor* x = &xs[base + j];
      if (!is_dense(x)) return PFB_E_UNSUPPORTED;
      d.src[j] = static_cast<const uint8_t*>(x->data);
      d.off[j] = dst_offsets[base + j];
      d.bytes[j] = numel(x) * dtype_size(x->dtype);
      if (d.bytes[j] > most) most = d.bytes[j];
    }
    if (most == 0) continue;
    const int gx = grid_for((most + 15) / 16, 256, 2);
    launch(pack_kernel, dim3((unsigned)gx, (unsigned)m), 256, 0, s, d,
           static_cast<uint8_t*>(dst));
    if (int e = launch_status()) return e;
  }
  return 0;
}

// copy_many: several dense tensor copies in one launch (a device-resident
// loop's carried values written back into its static state each trip).

namespace pfb {
struct CopyDesc {
  const uint8_t* src[kMaxPack];
  uint8_t* dst[kMaxPack];
  int64_t bytes[kMaxPack];
};

__global__ void __launch_bounds__(256) copy_many_kernel(CopyDesc d) {
  pdl_enter();
  const int t = blockIdx.y;
  const uint8_t* s = d.src[t];
  uint8_t* o = d.dst[t];
  const int64_t nb = d.bytes[t];
  const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(o)) & 15) == 0;
  const int64_t n16 = vec ? nb / 16 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride)
    reinterpret_cast<int4*>(o)[i] = __ldg(reinterpret_cast<const int4*>(s) + i);
  for (int64_t i = 16 * n16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += stride)
    o[i] = s[i];
}
// copy_many + the predicated while's loop test: pair `any_pair` is the
// active mask (u8 bools); every block of that pair ORs its bytes into
// scratch[0], every block takes a ticket (scratch[1]) and the last one sets
// the CUDA-graph conditional to any(mask) and resets the scratch words for
// the next trip -- the write-back and the test in one launch
__global__ void __launch_bounds__(256) copy_many_cond_kernel(CopyDesc d, int any_pair,
                                                             cudaGraphConditionalHandle h,
                                                             unsigned long long* counter,
                                                             int* scratch) {
  pdl_enter();
  const int t = blockIdx.y;
  const uint8_t* s = d.src[t];
  uint8_t* o = d.dst[t];
  const int64_t nb = d.bytes[t];
  const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(o)) & 15) == 0;
  const int64_t n16 = vec ? nb / 16 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int any = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
    const int4 v = __ldg(reinterpret_cast<const int4*>(s) + i);
    reinterpret_cast<int4*>(o)[i] = v;
    any |= (v.x | v.y | v.z | v.w) != 0;
  }
  for (int64_t i = 16 * n16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += stride) {
    const uint8_t v = s[i];
    o[i] = v;
    any |= v != 0;
  }
  any = __syncthreads_or(t == any_pair && any);
  if (threadIdx.x == 0) {
    if (any) atomicOr(&scratch[0], 1);
    __threadfence();
    const unsigned total = gridDim.x * gridDim.y;
    if ((unsigned)atomicAdd(&scratch[1], 1) == total - 1) {
      __threadfence();
      const int flag = atomicOr(&scratch[0], 0);
      cudaGraphSetConditional(h, flag ? 1u : 0u);
      if (counter) *counter += 1;
      scratch[0] = 0;
      scratch[1] = 0;
    }
  }
}
}  // namespace pfb

extern "C" int pfb_copy_many_cond(int32_t n, const pfb_tensor* srcs, const pfb_tensor* dsts,
                                  int32_t any_pair, uint64_t handle, void* counter, void* scratch,
                                  void* stream) {
  if (n < 1 || n > kMaxPack || any_pair < 0 || any_pair >= n || scratch == nullptr)
    return PFB_E_ARG;
  if (srcs[any_pair].dtype != PFB_BOOL) return PFB_E_DTYPE;
  CopyDesc d = {};
  int64_t most = 0;
  for (int j = 0; j < n; ++j) {
    const pfb_tensor* x = &srcs[j];
    const pfb_tensor* y = &dsts[j];
    if (!is_dense(x) || !is_dense(y) || x->dtype != y->dtype || numel(x) != numel(y))
      return PFB_E_UNSUPPORTED;
    d.src[j] = static_cast<const uint8_t*>(x->data);
    d.dst[j] = static_cast<uint8_t*>(y->data);
    d.bytes[j] = numel(x) * dtype_size(x->dtype);
    if (d.bytes[j] > most) most = d.bytes[j];
  }
  const int gx = grid_for(most > 0 ? (most + 15) / 16 : 1, 256, 2);
  launch(copy_many_cond_kernel, dim3((unsigned)gx, (unsigned)n), 256, 0, as_stream(stream), d,
         (int)any_pair, (cudaGraphConditionalHandle)handle, (unsigned long long*)counter,
         (int*)scratch);
  return launch_status();
}

extern "C" int pfb_copy_many(int32_t n, const pfb_tensor* srcs, const pfb_tensor* dsts,
                             void* stream) {
  if (n < 0) return PFB_E_ARG;
  cudaStream_t s = as_stream(stream);
  for (int base = 0; base < n; base += kMaxPack) {
    CopyDesc d = {};
    const int m = n - base < kMaxPack ? n - base : kMaxPack;
    int64_t most = 0;
    for (int j = 0; j < m; ++j) {
      const pfb_tensor* x = &srcs[base + j];
      const pfb_tensor* y = &dsts[base + j];
      if (!is_dense(x) || !is_dense(y) || x->dtype != y->dtype || numel(x) != numel(y))
        return PFB_E_UNSUPPORTED;
      d.src[j] = static_cast<const uint8_t*>(x->data);
      d.dst[j] = static_cast<uint8_t*>(y->data);
      d.bytes[j] = numel(x) * dtype_size(x->dtype);
      if (d.bytes[j] > most) most = d.bytes[j];
    }
    if (most == 0) continue;
    const int gx = grid_for((most + 15) / 16, 256, 2);
    launch(copy_many_kernel, dim3((unsigned)gx, (unsigned)m), 256, 0, s, d);
    if (int e = launch_status()) return e;
  }
  return 0;
}

// kernels this library has launched so far in the process (graph captures
// included: a captured launch is counted once, when recorded)
extern "C" int64_t pfb_kernel_launches(void) { return pfb::kernel_launches().load(); }
