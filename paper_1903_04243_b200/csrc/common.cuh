// Shared helpers for the libpfb kernels (sm_100a).
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdlib.h>

#include <utility>

#include "../../include/pfb.h"

namespace pfb {

constexpr int kMaxRank = PFB_MAX_RANK;
constexpr int kNumSMs = 148;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

inline int dtype_size(int dt) { return dt == PFB_F32 ? 4 : (dt == PFB_I64 ? 8 : 1); }

inline int64_t numel(const pfb_tensor* t) {
  int64_t n = 1;
  for (int i = 0; i < t->rank; ++i) n *= t->shape[i];
  return n;
}

inline bool is_dense(const pfb_tensor* t) {
  int64_t expect = 1;
  for (int i = t->rank - 1; i >= 0; --i) {
    if (t->shape[i] != 1 && t->stride[i] != expect) return false;
    expect *= t->shape[i];
  }
  return true;
}

// A set of up to N operands over one logical iteration shape, with dims of
// size 1 dropped and adjacent dims merged wherever every operand allows it.
// Operand 0 is conventionally the output.  `Layout` (9 operands) serves the
// elementwise / index kernels, `FLayout` (17) the fused programs.
constexpr int kMaxOps = 9;
constexpr int kMaxFOps = 17;
template <int N>
struct LayoutT {
  int rank;
  int nops;
  int64_t shape[kMaxRank];
  int64_t st[N][kMaxRank];
};
using Layout = LayoutT<kMaxOps>;
using FLayout = LayoutT<kMaxFOps>;

template <int N = kMaxOps>
inline LayoutT<N> make_layout(int rank, const int64_t* shape, int nops,
                              const int64_t* const* strides) {
  LayoutT<N> L;
  L.nops = nops;
  int r = 0;
  for (int d = 0; d < rank; ++d) {
    if (shape[d] == 1) continue;
    L.shape[r] = shape[d];
    for (int o = 0; o < nops; ++o) L.st[o][r] = strides[o][d];
    ++r;
  }
  // merge dim d into d-1 when st[d-1] == st[d] * shape[d] for all operands
  int w = 0;
  for (int d = 0; d < r; ++d) {
    if (w > 0) {
      bool ok = true;
      for (int o = 0; o < nops; ++o)
        if (L.st[o][w - 1] != L.st[o][d] * L.shape[d]) { ok = false; break; }
      if (ok) {
        L.shape[w - 1] *= L.shape[d];
        for (int o = 0; o < nops; ++o) L.st[o][w - 1] = L.st[o][d];
        continue;
      }
    }
    L.shape[w] = L.shape[d];
    for (int o = 0; o < nops; ++o) L.st[o][w] = L.st[o][d];
    ++w;
  }
  L.rank = w;
  if (w == 0) {  // scalar
    L.rank = 1;
    L.shape[0] = 1;
    for (int o = 0; o < nops; ++o) L.st[o][0] = 1;
  }
  return L;
}

// Right-align `t` to `rank` dims of `shape` with broadcasting; returns false
// when a dim is neither equal nor 1.
inline bool broadcast_strides(const pfb_tensor* t, int rank, const int64_t* shape, int64_t* st) {
  int off = rank - t->rank;
  if (off < 0) return false;
  for (int d = 0; d < rank; ++d) {
    if (d < off) { st[d] = 0; continue; }
    int64_t s = t->shape[d - off];
    if (s == shape[d]) st[d] = (s == 1) ? 0 : t->stride[d - off];
    else if (s == 1) st[d] = 0;
    else return false;
  }
  return true;
}

inline int grid_for(int64_t work, int block, int max_waves = 16) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * max_waves;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// --- device-side helpers -----------------------------------------------------

// offsets of element `lin` (row-major over L.shape) for the first NOPS operands
template <typename IdxT, int NOPS, int N>
__device__ __forceinline__ void offsets(const LayoutT<N>& L, IdxT lin, int64_t* off) {
  if (L.rank == 1) {  // collapsed to one dim (dense / scalar-broadcast operands): no division
#pragma unroll
    for (int o = 0; o < NOPS; ++o) off[o] = (int64_t)lin * L.st[o][0];
    return;
  }
#pragma unroll
  for (int o = 0; o < NOPS; ++o) off[o] = 0;
  for (int d = L.rank - 1; d >= 0; --d) {
    IdxT s = (IdxT)L.shape[d];
    IdxT q = lin / s;
    IdxT c = lin - q * s;
    lin = q;
#pragma unroll
    for (int o = 0; o < NOPS; ++o) off[o] += (int64_t)c * L.st[o][d];
  }
}

// Programmatic dependent launch: every kernel waits for its predecessor's
// memory at entry (griddepcontrol.wait) and immediately lets its successor
// start launching (launch_dependents), so back-to-back small kernels overlap
// their launch latency -- they are captured as programmatic edges in the CUDA
// graphs the executor replays.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

inline bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] == '1';
}

inline bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("PFB_DISABLE_PDL");
    return (e && e[0] == '1') ? 0 : 1;
  }();
  return on;
}

// kernels launched by this library (every launch site bumps it; the
// executor reports the difference across a run or a graph capture)
inline std::atomic<long long>& kernel_launches() {
  static std::atomic<long long> n{0};
  return n;
}

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args&&... args) {
  kernel_launches()++;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ void set_err(int32_t* err, int32_t bits) {
  if (err) atomicOr(err, bits);
}

// numpy maximum/minimum semantics: NaN propagates (first NaN wins)
__device__ __forceinline__ float np_max(float a, float b) {
  return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b));
}
__device__ __forceinline__ float np_min(float a, float b) {
  return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b));
}

}  // namespace pfb
