// Elementwise family: binary / unary / cast / strided copy / fill / fused
// programs.  Replaces reference tensor.py:104-188 and the layout copies of
// tensor.py:286-416.
//
// Loop-invariant operands arrive as stride-0 views (no materialised tile),
// so e.g. [320,32,256] * [32,256] reads the invariant once per row from L2.
// HBM-bound: 128-bit loads/stores on the inner dim whenever the operand is
// unit-stride and 16-byte aligned; index math in 32 bits when it fits.
#include "common.cuh"
#include "fused.cuh"

#include <algorithm>

namespace pfb {

// ----------------------------------------------------------------------------
// scalar op semantics (numpy-compatible)

template <int OP>
__device__ __forceinline__ float bin_f32(float a, float b) {
  if (OP == PFB_ADD) return a + b;
  if (OP == PFB_SUB) return a - b;
  if (OP == PFB_MUL) return a * b;
  if (OP == PFB_DIV) return a / b;           // IEEE: x/0 -> inf, 0/0 -> nan
  if (OP == PFB_MAX) return np_max(a, b);
  if (OP == PFB_MIN) return np_min(a, b);
  if (OP == PFB_LESS) return a < b ? 1.f : 0.f;
  return a == b ? 1.f : 0.f;
}

template <int OP>
__device__ __forceinline__ int64_t bin_i64(int64_t a, int64_t b) {
  // two's-complement wraparound like numpy int64
  uint64_t ua = (uint64_t)a, ub = (uint64_t)b;
  if (OP == PFB_ADD) return (int64_t)(ua + ub);
  if (OP == PFB_SUB) return (int64_t)(ua - ub);
  if (OP == PFB_MUL) return (int64_t)(ua * ub);
  if (OP == PFB_MAX) return a >= b ? a : b;
  if (OP == PFB_MIN) return a <= b ? a : b;
  if (OP == PFB_LESS) return a < b;
  return a == b;
}

template <int OP>
__device__ __forceinline__ float un_f32(float x) {
  if (OP == PFB_NEG) return -x;
  if (OP == PFB_EXP) return expf(x);
  if (OP == PFB_LOG) return logf(x);
  if (OP == PFB_RELU) return np_max(x, 0.f);
  if (OP == PFB_TANH) return tanhf(x);
  if (OP == PFB_SIGMOID) return 1.f / (1.f + expf(-x));
  if (OP == PFB_SQUARE) return x * x;
  return x == 0.f ? 1.f : 0.f;  // logical_not on 0/1 floats (fused programs)
}

template <int OP>
__device__ __forceinline__ int64_t un_i64(int64_t x) {
  if (OP == PFB_NEG) return (int64_t)(0ull - (uint64_t)x);
  if (OP == PFB_RELU) return x > 0 ? x : 0;
  return (int64_t)((uint64_t)x * (uint64_t)x);  // square
}

// Functors (Tin -> Tout), one template parameter per op so every op
// compiles to straight-line code.
template <int OP, bool CMP> struct BinF32 {
  __device__ __forceinline__ auto operator()(float a, float b) const {
    if constexpr (CMP) return (uint8_t)(bin_f32<OP>(a, b) != 0.f);
    else return bin_f32<OP>(a, b);
  }
};
template <int OP, bool CMP> struct BinI64 {
  __device__ __forceinline__ auto operator()(int64_t a, int64_t b) const {
    if constexpr (CMP) return (uint8_t)bin_i64<OP>(a, b);
    else return bin_i64<OP>(a, b);
  }
};
template <int OP> struct BinBool {
  __device__ __forceinline__ uint8_t operator()(uint8_t a, uint8_t b) const {
    return OP == PFB_LESS ? (uint8_t)(a < b) : (uint8_t)(a == b);
  }
};
template <int OP> struct UnF32 {
  __device__ __forceinline__ float operator()(float x, float) const { return un_f32<OP>(x); }
};
template <int OP> struct UnI64 {
  __device__ __forceinline__ int64_t operator()(int64_t x, int64_t) const { return un_i64<OP>(x); }
};
struct NotBool {
  __device__ __forceinline__ uint8_t operator()(uint8_t x, uint8_t) const { return x ? 0 : 1; }
};
template <typename Tin, typename Tout> struct Convert {
  __device__ __forceinline__ Tout operator()(Tin x, Tin) const {
    if constexpr (std::is_same<Tout, uint8_t>::value) return (uint8_t)(x != (Tin)0);
    else if constexpr (std::is_same<Tin, float>::value && std::is_same<Tout, int64_t>::value) {
      // truncation toward zero; numpy gives INT64_MIN for nan / out of range
      if (!(x >= -9.2233720368547758e18f && x < 9.2233720368547758e18f)) return INT64_MIN;
      return (int64_t)x;
    } else return (Tout)x;
  }
};
template <typename T> struct Identity {
  __device__ __forceinline__ T operator()(T x, T) const { return x; }
};

// ----------------------------------------------------------------------------
// vector helpers: 4 consecutive elements along the inner dim

template <typename T>
__device__ __forceinline__ void load4(const T* p, int64_t st, bool vec, T* v) {
  if (st == 0) {
    T x = __ldg(p);
    v[0] = v[1] = v[2] = v[3] = x;
  } else if (vec) {
    if constexpr (sizeof(T) == 4) {
      float4 t = __ldg(reinterpret_cast<const float4*>(p));
      const T* q = reinterpret_cast<const T*>(&t);
      v[0] = q[0]; v[1] = q[1]; v[2] = q[2]; v[3] = q[3];
    } else if constexpr (sizeof(T) == 8) {
      const longlong2* w = reinterpret_cast<const longlong2*>(p);
      longlong2 t0 = __ldg(w), t1 = __ldg(w + 1);
      v[0] = (T)t0.x; v[1] = (T)t0.y; v[2] = (T)t1.x; v[3] = (T)t1.y;
    } else {
      uchar4 t = __ldg(reinterpret_cast<const uchar4*>(p));
      v[0] = (T)t.x; v[1] = (T)t.y; v[2] = (T)t.z; v[3] = (T)t.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldg(p + k * st);
  }
}

template <typename T>
__device__ __forceinline__ void store4(T* p, int64_t st, bool vec, const T* v) {
  if (vec) {
    if constexpr (sizeof(T) == 4) {
      float4 t;
      T* q = reinterpret_cast<T*>(&t);
      q[0] = v[0]; q[1] = v[1]; q[2] = v[2]; q[3] = v[3];
      *reinterpret_cast<float4*>(p) = t;
    } else if constexpr (sizeof(T) == 8) {
      longlong2* w = reinterpret_cast<longlong2*>(p);
      w[0] = make_longlong2((long long)v[0], (long long)v[1]);
      w[1] = make_longlong2((long long)v[2], (long long)v[3]);
    } else {
      *reinterpret_cast<uchar4*>(p) = make_uchar4(v[0], v[1], v[2], v[3]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k * st] = v[k];
  }
}

// Grid-stride kernels.  Operand 0 of the layout is the output, 1..NIN inputs.
template <typename Tin, typename Tout, typename F, typename IdxT, int NIN>
__global__ void __launch_bounds__(256) ew_vec4_kernel(Layout L, IdxT nchunks, Tout* out,
                                                      const Tin* a, const Tin* b, F f,
                                                      unsigned vecmask) {
  pdl_enter();
  const int last = L.rank - 1;
  const int64_t so = L.st[0][last], sa = L.st[1][last], sb = NIN > 1 ? L.st[2][last] : 0;
  // U grid-stride chunks per trip: all U chunks' loads are issued before any
  // is consumed (U x 16 bytes in flight per thread and input; U = 4 for
  // byte-sized outputs, whose stores are only 4 bytes per thread)
  constexpr int U = sizeof(Tout) == 1 ? 4 : 2;
  const IdxT S = (IdxT)gridDim.x * blockDim.x;
  for (IdxT c = blockIdx.x * (IdxT)blockDim.x + threadIdx.x; c < nchunks; c += U * S) {
    int64_t off[U][NIN + 1];
    Tin x[U][4], y[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u == 0 || c + u * S < nchunks) {
        offsets<IdxT, NIN + 1>(L, (c + u * S) * 4, off[u]);
        load4(a + off[u][1], sa, vecmask & 2u, x[u]);
        if (NIN > 1) load4(b + off[u][2], sb, vecmask & 4u, y[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u == 0 || c + u * S < nchunks) {
        Tout r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = f(x[u][k], NIN > 1 ? y[u][k] : x[u][k]);
        store4(out + off[u][0], so, vecmask & 1u, r);
      }
    }
  }
}

template <typename Tin, typename Tout, typename F, typename IdxT, int NIN>
__global__ void __launch_bounds__(256) ew_scalar_kernel(Layout L, IdxT n, Tout* out,
                                                        const Tin* a, const Tin* b, F f) {
  pdl_enter();
  for (IdxT i = blockIdx.x * (IdxT)blockDim.x + threadIdx.x; i < n;
       i += (IdxT)gridDim.x * blockDim.x) {
    int64_t off[NIN + 1];
    offsets<IdxT, NIN + 1>(L, i, off);
    Tin x = a[off[1]];
    out[off[0]] = f(x, NIN > 1 ? b[off[2]] : x);
  }
}

// One-input op whose input is transposed relative to its output (a
// materialised transpose, or a unary / cast of one): 32x32 tiles through
// shared memory over (p, last), p = the input's unit-stride dim, so both the
// input reads (lanes along p) and the output writes (lanes along last) are
// coalesced.  Other dims are the batch (blockIdx.y, grid-stride).
template <typename Tin, typename Tout, typename F>
__global__ void __launch_bounds__(256) ew_tile_transpose(Layout L, int p, int64_t nbatch,
                                                         int64_t tiles_last, Tout* out,
                                                         const Tin* in, F f) {
  pdl_enter();
  // a block owns two adjacent 32x32 tiles along `last` (the loads of both are
  // in flight before the exchange)
  __shared__ Tin t[2][32][33];
  const int last = L.rank - 1;
  const int64_t tl = 2 * (blockIdx.x % tiles_last), tp = blockIdx.x / tiles_last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t np = L.shape[p], nl = L.shape[last];
  const int64_t isp = L.st[1][p], isl = L.st[1][last], osp = L.st[0][p], osl = L.st[0][last];
  // interior tiles: no bounds checks, addresses advance by hoisted strides
  const bool full = (tp + 1) * 32 <= np && (tl + 2) * 32 <= nl;
  for (int64_t bi = blockIdx.y; bi < nbatch; bi += gridDim.y) {
    int64_t ob = 0, ib = 0;
    if (L.rank > 2) {
      int64_t rem = bi;
      for (int d = last; d >= 0; --d) {
        if (d == p || d == last) continue;
        const int64_t c = rem % L.shape[d];
        rem /= L.shape[d];
        ob += c * L.st[0][d];
        ib += c * L.st[1][d];
      }
    }
    const Tin* src = in + ib + (tp * 32 + tx) * isp + (tl * 32 + ty) * isl;
    Tout* dst = out + ob + (tp * 32 + ty) * osp + (tl * 32 + tx) * osl;
    if (full) {
      Tin v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(src + u * 8 * isl);
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u >> 2][ty + 8 * (u & 3)][tx] = v[u];
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const Tin x = t[u >> 2][tx][ty + 8 * (u & 3)];
        dst[(u & 3) * 8 * osp + (u >> 2) * 32 * osl] = f(x, x);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = ty + 8 * (u & 3) + 32 * (u >> 2);
        if (tp * 32 + tx < np && tl * 32 + j < nl) t[u >> 2][j & 31][tx] = src[(j - ty) * isl];
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = ty + 8 * (u & 3);
        const int64_t il = tl * 32 + 32 * (u >> 2) + tx;
        if (tp * 32 + j < np && il < nl) {
          const Tin x = t[u >> 2][tx][j];
          dst[(u & 3) * 8 * osp + (u >> 2) * 32 * osl] = f(x, x);
        }
      }
    }
    __syncthreads();
  }
}

// Host launcher: `L` over (out, a[, b]); picks the vector path when the inner
// dim allows it.
template <typename Tin, typename Tout, int NIN, typename F>
int launch_ew(const Layout& L, void* out, const void* a, const void* b, F f, cudaStream_t s) {
  int64_t n = 1;
  for (int d = 0; d < L.rank; ++d) n *= L.shape[d];
  if (n == 0) return 0;
  const int last = L.rank - 1;
  if (NIN == 1 && L.rank >= 2 && L.st[0][last] == 1 && L.st[1][last] != 1 && n >= 4096) {
    int p = -1;
    for (int d = 0; d < last; ++d)
      if (L.st[1][d] == 1 && L.shape[d] > 1) p = d;
    if (p >= 0) {
      const int64_t tiles_last = (L.shape[last] + 63) / 64, tiles_p = (L.shape[p] + 31) / 32;
      int64_t nbatch = n / (L.shape[last] * L.shape[p]);
      if (tiles_last * tiles_p <= 0x7fffffff) {
        const unsigned gy = (unsigned)std::min<int64_t>(nbatch, 65535);
        launch(ew_tile_transpose<Tin, Tout, F>, dim3((unsigned)(tiles_last * tiles_p), gy), 256,
               0, s, L, p, nbatch, tiles_last, (Tout*)out, (const Tin*)a, f);
        return launch_status();
      }
    }
  }
  bool vec_dim = (L.shape[last] % 4) == 0;
  unsigned vecmask = 0;
  if (vec_dim) {
    const void* ptrs[3] = {out, a, b};
    for (int o = 0; o <= NIN; ++o) {
      size_t esz = o == 0 ? sizeof(Tout) : sizeof(Tin);
      bool ok = L.st[o][last] == 1 && ((uintptr_t)ptrs[o] % (4 * esz)) == 0;
      for (int d = 0; d < last && ok; ++d) ok = (L.st[o][d] % 4) == 0;
      if (ok) vecmask |= 1u << o;
    }
  }
  const int block = 256;
  bool small = n < (int64_t)0x7fffffff;
  if (vec_dim) {
    int64_t chunks = n / 4;
    int grid = grid_for(chunks, block);
    if (small)
      launch(ew_vec4_kernel<Tin, Tout, F, uint32_t, NIN>, grid, block, 0, s, 
          L, (uint32_t)chunks, (Tout*)out, (const Tin*)a, (const Tin*)b, f, vecmask);
    else
      launch(ew_vec4_kernel<Tin, Tout, F, int64_t, NIN>, grid, block, 0, s, 
          L, chunks, (Tout*)out, (const Tin*)a, (const Tin*)b, f, vecmask);
  } else {
    int grid = grid_for(n, block);
    if (small)
      launch(ew_scalar_kernel<Tin, Tout, F, uint32_t, NIN>, grid, block, 0, s, 
          L, (uint32_t)n, (Tout*)out, (const Tin*)a, (const Tin*)b, f);
    else
      launch(ew_scalar_kernel<Tin, Tout, F, int64_t, NIN>, grid, block, 0, s, 
          L, n, (Tout*)out, (const Tin*)a, (const Tin*)b, f);
  }
  return launch_status();
}

// Build the (out, in...) layout with numpy broadcasting of inputs to out.
inline int ew_layout(pfb_tensor* out, const pfb_tensor* a, const pfb_tensor* b, Layout* L) {
  int64_t sa[kMaxRank], sb[kMaxRank];
  if (!broadcast_strides(a, out->rank, out->shape, sa)) return PFB_E_SHAPE;
  if (b && !broadcast_strides(b, out->rank, out->shape, sb)) return PFB_E_SHAPE;
  const int64_t* st[3] = {out->stride, sa, sb};
  *L = make_layout(out->rank, out->shape, b ? 3 : 2, st);
  return 0;
}

template <int OP>
int binary_dispatch(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out, cudaStream_t s) {
  Layout L;
  if (int e = ew_layout(out, a, b, &L)) return e;
  constexpr bool CMP = OP == PFB_LESS || OP == PFB_EQUAL;
  switch (a->dtype) {
    case PFB_F32:
      if (out->dtype != (CMP ? PFB_BOOL : PFB_F32)) return PFB_E_DTYPE;
      return launch_ew<float, typename std::conditional<CMP, uint8_t, float>::type, 2>(
          L, out->data, a->data, b->data, BinF32<OP, CMP>{}, s);
    case PFB_I64:
      if (OP == PFB_DIV) return PFB_E_DTYPE;
      if (out->dtype != (CMP ? PFB_BOOL : PFB_I64)) return PFB_E_DTYPE;
      return launch_ew<int64_t, typename std::conditional<CMP, uint8_t, int64_t>::type, 2>(
          L, out->data, a->data, b->data, BinI64<OP, CMP>{}, s);
    default:
      if (!CMP || out->dtype != PFB_BOOL) return PFB_E_DTYPE;
      return launch_ew<uint8_t, uint8_t, 2>(L, out->data, a->data, b->data, BinBool<OP>{}, s);
  }
}

template <int OP>
int unary_dispatch(const pfb_tensor* x, pfb_tensor* out, cudaStream_t s) {
  Layout L;
  if (int e = ew_layout(out, x, nullptr, &L)) return e;
  if (x->dtype != out->dtype) return PFB_E_DTYPE;
  if (OP == PFB_LOGICAL_NOT) {
    if (x->dtype != PFB_BOOL) return PFB_E_DTYPE;
    return launch_ew<uint8_t, uint8_t, 1>(L, out->data, x->data, nullptr, NotBool{}, s);
  }
  if (x->dtype == PFB_F32)
    return launch_ew<float, float, 1>(L, out->data, x->data, nullptr, UnF32<OP>{}, s);
  if (x->dtype == PFB_I64 && (OP == PFB_NEG || OP == PFB_RELU || OP == PFB_SQUARE))
    return launch_ew<int64_t, int64_t, 1>(L, out->data, x->data, nullptr, UnI64<OP>{}, s);
  return PFB_E_DTYPE;
}

template <typename Tin>
int cast_from(const Layout& L, const pfb_tensor* x, pfb_tensor* out, cudaStream_t s) {
  switch (out->dtype) {
    case PFB_F32:
      return launch_ew<Tin, float, 1>(L, out->data, x->data, nullptr, Convert<Tin, float>{}, s);
    case PFB_I64:
      return launch_ew<Tin, int64_t, 1>(L, out->data, x->data, nullptr, Convert<Tin, int64_t>{}, s);
    default:
      return launch_ew<Tin, uint8_t, 1>(L, out->data, x->data, nullptr, Convert<Tin, uint8_t>{}, s);
  }
}

// ----------------------------------------------------------------------------
// fused elementwise programs (float registers; bool inputs read as 0/1)

// One templated kernel for both widths: V = 4 runs the program on 4
// consecutive elements of the innermost dim per thread (extent a multiple of
// 4; contiguous operands move as 128-bit accesses), V = 1 on single elements.
// The program is staged in shared memory once per CTA; each step is one
// warp-uniform switch whose cases apply the op to all V lanes, so dispatch,
// offset arithmetic and register-file traffic are paid once per V elements.
// Operand feed modes (2 bits per operand, operand 0 = output): 0 = contiguous
// + aligned vector, 1 = inner-dim broadcast, 2 = strided.
template <int V>
struct alignas(4 * V) Vec {
  float v[V];
};

template <int V, typename T>
__device__ __forceinline__ Vec<V> load_v(const void* base, int64_t off, int64_t inner, int mode) {
  Vec<V> r;
  const T* p = reinterpret_cast<const T*>(base) + off;
  if (V == 4 && mode == 0) {
    if constexpr (std::is_same<T, float>::value) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(p));
      r.v[0] = f.x; r.v[1] = f.y; r.v[2] = f.z; r.v[3] = f.w;
    } else {
      const uchar4 u = __ldg(reinterpret_cast<const uchar4*>(p));
      r.v[0] = u.x; r.v[1] = u.y; r.v[2] = u.z; r.v[3] = u.w;
    }
    return r;
  }
  if (mode == 1) {
    const float x = (float)__ldg(p);
#pragma unroll
    for (int j = 0; j < V; ++j) r.v[j] = x;
    return r;
  }
#pragma unroll
  for (int j = 0; j < V; ++j) r.v[j] = (float)__ldg(p + j * inner);
  return r;
}

#define PFB_EW1(EXPR)                                     \
  {                                                       \
    _Pragma("unroll") for (int j = 0; j < V; ++j) {       \
      const float x = a.v[j];                             \
      (void)x;                                            \
      o.v[j] = (EXPR);                                    \
    }                                                     \
  }                                                       \
  break;
#define PFB_EW2(EXPR)                                     \
  {                                                       \
    _Pragma("unroll") for (int j = 0; j < V; ++j) {       \
      const float x = a.v[j], y = b.v[j];                 \
      o.v[j] = (EXPR);                                    \
    }                                                     \
  }                                                       \
  break;

template <int V>
__device__ __forceinline__ void store_v(void* base, int dt, int64_t off, int64_t inner, bool vec,
                                        const Vec<V>& res) {
  if (dt == PFB_BOOL) {
    uint8_t* q = reinterpret_cast<uint8_t*>(base) + off;
    if (V == 4 && vec) {
      *reinterpret_cast<uchar4*>(q) = make_uchar4(res.v[0] != 0.f, res.v[1] != 0.f,
                                                  res.v[V > 2 ? 2 : 0] != 0.f,
                                                  res.v[V > 3 ? 3 : 0] != 0.f);
      return;
    }
#pragma unroll
    for (int j = 0; j < V; ++j) q[j * inner] = (uint8_t)(res.v[j] != 0.f);
  } else {
    float* q = reinterpret_cast<float*>(base) + off;
    if (V == 4 && vec) {
      *reinterpret_cast<float4*>(q) = make_float4(res.v[0], res.v[V > 1 ? 1 : 0],
                                                  res.v[V > 2 ? 2 : 0], res.v[V > 3 ? 3 : 0]);
      return;
    }
#pragma unroll
    for (int j = 0; j < V; ++j) q[j * inner] = res.v[j];
  }
}

// NIN: input slots compiled in (2 / 4 / 8 / 16, >= P.n_in)
template <typename IdxT, int NIN, int V>
__global__ void __launch_bounds__(256) fused_kernel(FLayout L, IdxT ngroups, FusedProgram P,
                                                    FeedModes modes, FusedOuts outs,
                                                    FusedIns ins) {
  pdl_enter();
  __shared__ int4 prog[kMaxSteps];
  for (int s = threadIdx.x; s < P.n_steps; s += blockDim.x)
    prog[s] = make_int4(P.code[s][0], P.code[s][1], P.code[s][2], P.code[s][3]);
  __syncthreads();
  const int nsteps = P.n_steps;
  const int ir = L.rank - 1;
  for (IdxT g = blockIdx.x * (IdxT)blockDim.x + threadIdx.x; g < ngroups;
       g += (IdxT)gridDim.x * blockDim.x) {
    int64_t off[NIN + 1];
    offsets<IdxT, NIN + 1>(L, g * V, off);
    // every input is loaded up front, all loads in flight together (a load
    // step of the program then only moves a register): the interpreter's
    // register file lives in local memory, and loading inside the step loop
    // serialised one memory latency per input
    Vec<V> in[NIN];
#pragma unroll
    for (int K = 0; K < NIN; ++K) {
      if (K >= P.n_in) break;
      const int md = (int)((modes >> (2 * (K + 1))) & 3);
      in[K] = P.in_dtype[K] == PFB_BOOL
                  ? load_v<V, uint8_t>(ins.p[K], off[K + 1], L.st[K + 1][ir], md)
                  : load_v<V, float>(ins.p[K], off[K + 1], L.st[K + 1][ir], md);
    }
    Vec<V> r[kMaxRegs];
    for (int s = 0; s < nsteps; ++s) {
      const int4 c = prog[s];
      Vec<V> o;
      if (c.x == F_LOAD) {
        switch (c.z) {
#define PFB_LD(K)                     \
  case K:                             \
    if (K < NIN) o = in[K < NIN ? K : 0]; \
    break;
          PFB_LD(0) PFB_LD(1) PFB_LD(2) PFB_LD(3) PFB_LD(4) PFB_LD(5) PFB_LD(6) PFB_LD(7)
          PFB_LD(8) PFB_LD(9) PFB_LD(10) PFB_LD(11) PFB_LD(12) PFB_LD(13) PFB_LD(14) PFB_LD(15)
#undef PFB_LD
        }
      } else if (c.x == F_CONST) {
        const float x = __int_as_float(c.z);
#pragma unroll
        for (int j = 0; j < V; ++j) o.v[j] = x;
      } else if (c.x == F_SELECT) {
        const Vec<V> pr = r[c.z], t = r[c.w], e = r[c.y];
#pragma unroll
        for (int j = 0; j < V; ++j) o.v[j] = pr.v[j] != 0.f ? t.v[j] : e.v[j];
      } else {
        const Vec<V> a = r[c.z];
        const Vec<V> b = r[c.w];
        switch (c.x) {
          case PFB_ADD: PFB_EW2(x + y)
          case PFB_SUB: PFB_EW2(x - y)
          case PFB_MUL: PFB_EW2(x * y)
          case PFB_DIV: PFB_EW2(x / y)
          case PFB_MAX: PFB_EW2(np_max(x, y))
          case PFB_MIN: PFB_EW2(np_min(x, y))
          case PFB_LESS: PFB_EW2(x < y ? 1.f : 0.f)
          case PFB_EQUAL: PFB_EW2(x == y ? 1.f : 0.f)
          case 16 + PFB_NEG: PFB_EW1(-x)
          case 16 + PFB_EXP: PFB_EW1(expf(x))
          case 16 + PFB_LOG: PFB_EW1(logf(x))
          case 16 + PFB_RELU: PFB_EW1(np_max(x, 0.f))
          case 16 + PFB_TANH: PFB_EW1(tanhf(x))
          case 16 + PFB_SIGMOID: PFB_EW1(1.f / (1.f + expf(-x)))
          case 16 + PFB_SQUARE: PFB_EW1(x * x)
          case 16 + PFB_LOGICAL_NOT: PFB_EW1(x == 0.f ? 1.f : 0.f)
          case 66: PFB_EW1(x != 0.f ? 1.f : 0.f)  // cast f32 -> bool
          default: o = a; break;                  // 67: move (cast bool -> f32)
        }
      }
      r[c.y] = o;
    }
    // outputs share one dense layout: operand 0's offsets
    const bool vec = (modes & 3) == 0;
    for (int k = 0; k < P.n_out; ++k)
      store_v<V>(outs.p[k], P.out_dt[k], off[0], L.st[0][ir], vec, r[P.out_reg[k]]);
  }
}
#undef PFB_EW1
#undef PFB_EW2

template <int V, typename IdxT>
void launch_fused(int n_in, const FLayout& L, IdxT ngroups, const FusedProgram& P,
                  FeedModes modes, const FusedOuts& outs, const FusedIns& ins, cudaStream_t s) {
  const int grid = grid_for((int64_t)ngroups, 256);
  if (n_in <= 2) launch(fused_kernel<IdxT, 2, V>, grid, 256, 0, s, L, ngroups, P, modes, outs, ins);
  else if (n_in <= 4) launch(fused_kernel<IdxT, 4, V>, grid, 256, 0, s, L, ngroups, P, modes, outs, ins);
  else if (n_in <= 8) launch(fused_kernel<IdxT, 8, V>, grid, 256, 0, s, L, ngroups, P, modes, outs, ins);
  else launch(fused_kernel<IdxT, 16, V>, grid, 256, 0, s, L, ngroups, P, modes, outs, ins);
}

// ---------------------------------------------------------------------------
// Integer-domain fused programs (F3 over i64 / bool: loop counters, index
// arithmetic, masks of predicated control flow).  Same program encoding as
// the float interpreter; registers are int64 (bool = 0/1), i64 wraps like
// numpy; constants are int32 immediates.  One element per thread (these
// tensors are [n]-sized bookkeeping values).
template <typename IdxT, int NIN>
__global__ void __launch_bounds__(256) fused_int_kernel(FLayout L, IdxT n, FusedProgram P,
                                                        FusedOuts outs, FusedIns ins) {
  pdl_enter();
  __shared__ int4 prog[kMaxSteps];
  for (int s = threadIdx.x; s < P.n_steps; s += blockDim.x)
    prog[s] = make_int4(P.code[s][0], P.code[s][1], P.code[s][2], P.code[s][3]);
  __syncthreads();
  for (IdxT e = blockIdx.x * (IdxT)blockDim.x + threadIdx.x; e < n;
       e += (IdxT)gridDim.x * blockDim.x) {
    int64_t off[NIN + 1];
    offsets<IdxT, NIN + 1>(L, e, off);
    int64_t in[NIN];
#pragma unroll
    for (int K = 0; K < NIN; ++K) {
      if (K >= P.n_in) break;
      in[K] = P.in_dtype[K] == PFB_BOOL
                  ? (int64_t)__ldg(reinterpret_cast<const uint8_t*>(ins.p[K]) + off[K + 1])
                  : __ldg(reinterpret_cast<const long long*>(ins.p[K]) + off[K + 1]);
    }
    int64_t r[kMaxRegs];
    for (int s = 0; s < P.n_steps; ++s) {
      const int4 c = prog[s];
      int64_t o = 0;
      if (c.x == F_LOAD) {
        switch (c.z) {
#define PFB_LDI(K) case K: if (K < NIN) o = in[K < NIN ? K : 0]; break;
          PFB_LDI(0) PFB_LDI(1) PFB_LDI(2) PFB_LDI(3) PFB_LDI(4) PFB_LDI(5) PFB_LDI(6) PFB_LDI(7)
          PFB_LDI(8) PFB_LDI(9) PFB_LDI(10) PFB_LDI(11) PFB_LDI(12) PFB_LDI(13) PFB_LDI(14)
          PFB_LDI(15)
#undef PFB_LDI
        }
      } else if (c.x == F_CONST) {
        o = (int64_t)c.z;
      } else if (c.x == F_SELECT) {
        o = r[c.z] != 0 ? r[c.w] : r[c.y];
      } else {
        const int64_t a = r[c.z], b = r[c.w];
        const uint64_t ua = (uint64_t)a, ub = (uint64_t)b;
        switch (c.x) {
          case PFB_ADD: o = (int64_t)(ua + ub); break;
          case PFB_SUB: o = (int64_t)(ua - ub); break;
          case PFB_MUL: o = (int64_t)(ua * ub); break;
          case PFB_MAX: o = a >= b ? a : b; break;
          case PFB_MIN: o = a <= b ? a : b; break;
          case PFB_LESS: o = a < b; break;
          case PFB_EQUAL: o = a == b; break;
          case 16 + PFB_NEG: o = (int64_t)(0 - ua); break;
          case 16 + PFB_SQUARE: o = (int64_t)(ua * ua); break;
          case 16 + PFB_LOGICAL_NOT: o = a == 0; break;
          case 66: o = a != 0; break;  // to bool
          default: o = a; break;        // 67: move
        }
      }
      r[c.y] = o;
    }
    for (int k = 0; k < P.n_out; ++k) {
      const int64_t v = r[P.out_reg[k]];
      if (P.out_dt[k] == PFB_BOOL)
        reinterpret_cast<uint8_t*>(outs.p[k])[off[0]] = (uint8_t)(v != 0);
      else if (P.out_dt[k] == PFB_F32)  // the group's final cast to f64 (fp32 storage)
        reinterpret_cast<float*>(outs.p[k])[off[0]] = (float)v;
      else
        reinterpret_cast<long long*>(outs.p[k])[off[0]] = v;
    }
  }
}
}  // namespace pfb

using namespace pfb;

extern "C" int pfb_fused_int(int32_t n_in, const pfb_tensor* ins, int32_t n_steps,
                             const int32_t* program, int32_t n_out, const int32_t* out_regs,
                             pfb_tensor* outs, void* stream) {
  if (n_in < 1 || n_in > kMaxIn || n_steps < 1 || n_steps > kMaxSteps) return PFB_E_ARG;
  if (n_out < 1 || n_out > kMaxOuts) return PFB_E_ARG;
  const pfb_tensor* out = &outs[0];
  for (int k = 0; k < n_out; ++k) {
    if (outs[k].dtype != PFB_I64 && outs[k].dtype != PFB_BOOL && outs[k].dtype != PFB_F32)
      return PFB_E_DTYPE;
    if (outs[k].rank != out->rank) return PFB_E_SHAPE;
    for (int d = 0; d < out->rank; ++d)
      if (outs[k].shape[d] != out->shape[d] ||
          (out->shape[d] > 1 && outs[k].stride[d] != out->stride[d]))
        return PFB_E_SHAPE;
    if (out_regs[k] < 0 || out_regs[k] >= kMaxRegs) return PFB_E_ARG;
  }
  int64_t stb[kMaxIn][kMaxRank];
  const int64_t* st[kMaxFOps];
  st[0] = out->stride;
  FusedProgram P;
  P.n_in = n_in;
  P.n_steps = n_steps;
  for (int k = 0; k < n_in; ++k) {
    if (ins[k].dtype != PFB_I64 && ins[k].dtype != PFB_BOOL) return PFB_E_DTYPE;
    if (!broadcast_strides(&ins[k], out->rank, out->shape, stb[k])) return PFB_E_SHAPE;
    st[k + 1] = stb[k];
    P.in_dtype[k] = ins[k].dtype;
  }
  for (int k = n_in; k < kMaxIn; ++k) P.in_dtype[k] = PFB_I64;
  for (int s = 0; s < n_steps; ++s) {
    for (int j = 0; j < 4; ++j) P.code[s][j] = program[4 * s + j];
    if (P.code[s][1] < 0 || P.code[s][1] >= kMaxRegs) return PFB_E_ARG;
  }
  FusedOuts fo;
  P.n_out = n_out;
  for (int k = 0; k < kMaxOuts; ++k) {
    fo.p[k] = k < n_out ? outs[k].data : nullptr;
    P.out_reg[k] = k < n_out ? out_regs[k] : 0;
    P.out_dt[k] = k < n_out ? outs[k].dtype : PFB_I64;
  }
  FLayout L = make_layout<kMaxFOps>(out->rank, out->shape, n_in + 1, st);
  const int64_t n = numel(out);
  if (n == 0) return 0;
  FusedIns fi;
  for (int k = 0; k < kMaxIn; ++k) fi.p[k] = k < n_in ? ins[k].data : nullptr;
  cudaStream_t s = as_stream(stream);
  if (fused_int_jit_launch(P, n >= (int64_t)0x7fffffff, L, n, fo, fi, s)) return launch_status();
  const int grid = grid_for(n, 256);
  const bool small = n < (int64_t)0x7fffffff;
#define PFB_FI(K)                                                                              \
  if (small) launch(fused_int_kernel<uint32_t, K>, grid, 256, 0, s, L, (uint32_t)n, P, fo, fi); \
  else launch(fused_int_kernel<int64_t, K>, grid, 256, 0, s, L, n, P, fo, fi);
  if (n_in <= 4) { PFB_FI(4) }
  else if (n_in <= 8) { PFB_FI(8) }
  else { PFB_FI(16) }
#undef PFB_FI
  return launch_status();
}

extern "C" int pfb_binary(int32_t op, const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                          void* stream) {
  cudaStream_t s = as_stream(stream);
  if (a->dtype != b->dtype) return PFB_E_DTYPE;
  switch (op) {
    case PFB_ADD: return binary_dispatch<PFB_ADD>(a, b, out, s);
    case PFB_SUB: return binary_dispatch<PFB_SUB>(a, b, out, s);
    case PFB_MUL: return binary_dispatch<PFB_MUL>(a, b, out, s);
    case PFB_DIV: return binary_dispatch<PFB_DIV>(a, b, out, s);
    case PFB_MAX: return binary_dispatch<PFB_MAX>(a, b, out, s);
    case PFB_MIN: return binary_dispatch<PFB_MIN>(a, b, out, s);
    case PFB_LESS: return binary_dispatch<PFB_LESS>(a, b, out, s);
    case PFB_EQUAL: return binary_dispatch<PFB_EQUAL>(a, b, out, s);
    default: return PFB_E_ARG;
  }
}

extern "C" int pfb_unary(int32_t op, const pfb_tensor* x, pfb_tensor* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  switch (op) {
    case PFB_NEG: return unary_dispatch<PFB_NEG>(x, out, s);
    case PFB_EXP: return unary_dispatch<PFB_EXP>(x, out, s);
    case PFB_LOG: return unary_dispatch<PFB_LOG>(x, out, s);
    case PFB_RELU: return unary_dispatch<PFB_RELU>(x, out, s);
    case PFB_TANH: return unary_dispatch<PFB_TANH>(x, out, s);
    case PFB_SIGMOID: return unary_dispatch<PFB_SIGMOID>(x, out, s);
    case PFB_SQUARE: return unary_dispatch<PFB_SQUARE>(x, out, s);
    case PFB_LOGICAL_NOT: return unary_dispatch<PFB_LOGICAL_NOT>(x, out, s);
    default: return PFB_E_ARG;
  }
}

extern "C" int pfb_cast(const pfb_tensor* x, pfb_tensor* out, void* stream) {
  Layout L;
  if (int e = ew_layout(out, x, nullptr, &L)) return e;
  cudaStream_t s = as_stream(stream);
  switch (x->dtype) {
    case PFB_F32: return cast_from<float>(L, x, out, s);
    case PFB_I64: return cast_from<int64_t>(L, x, out, s);
    default: return cast_from<uint8_t>(L, x, out, s);
  }
}

extern "C" int pfb_copy(const pfb_tensor* x, pfb_tensor* out, void* stream) {
  if (x->dtype != out->dtype) return PFB_E_DTYPE;
  Layout L;
  if (int e = ew_layout(out, x, nullptr, &L)) return e;
  cudaStream_t s = as_stream(stream);
  switch (x->dtype) {
    case PFB_F32: return launch_ew<float, float, 1>(L, out->data, x->data, nullptr, Identity<float>{}, s);
    case PFB_I64:
      return launch_ew<int64_t, int64_t, 1>(L, out->data, x->data, nullptr, Identity<int64_t>{}, s);
    default:
      return launch_ew<uint8_t, uint8_t, 1>(L, out->data, x->data, nullptr, Identity<uint8_t>{}, s);
  }
}

namespace pfb {
template <typename T>
__global__ void fill_kernel(Layout L, int64_t n, T* out, T v) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t off[1];
    offsets<int64_t, 1>(L, i, off);
    out[off[0]] = v;
  }
}
}  // namespace pfb

extern "C" int pfb_fill(pfb_tensor* out, double value, void* stream) {
  const int64_t* st[1] = {out->stride};
  Layout L = make_layout(out->rank, out->shape, 1, st);
  int64_t n = numel(out);
  if (n == 0) return 0;
  cudaStream_t s = as_stream(stream);
  int grid = grid_for(n, 256);
  if (out->dtype == PFB_F32) launch(fill_kernel<float>, grid, 256, 0, s, L, n, (float*)out->data, (float)value);
  else if (out->dtype == PFB_I64) launch(fill_kernel<int64_t>, grid, 256, 0, s, L, n, (int64_t*)out->data, (int64_t)value);
  else launch(fill_kernel<uint8_t>, grid, 256, 0, s, L, n, (uint8_t*)out->data, (uint8_t)(value != 0.0));
  return launch_status();
}

static int fused_impl(int32_t n_in, const pfb_tensor* ins, int32_t n_steps,
                      const int32_t* program, int32_t n_out, const int32_t* out_regs,
                      pfb_tensor* outs, void* stream, const int64_t* parts = nullptr,
                      const int32_t* rowsum = nullptr) {
  if (n_in < 1 || n_in > kMaxIn || n_steps < 1 || n_steps > kMaxSteps) return PFB_E_ARG;
  int RS[kMaxIn];
  if (rowsum) {
    bool any = false;
    for (int k = 0; k < n_in; ++k) {
      // j | op << 16: the sum of input j (op: a unary program opcode applied
      // to it first, 0 = none)
      RS[k] = rowsum[k] < 0 ? -1 : rowsum[k];
      const int op = RS[k] < 0 ? 0 : RS[k] >> 16;
      if (RS[k] >= 0 && ((RS[k] & 0xffff) >= n_in || (op != 0 && (op < 16 || op > 16 + PFB_SQUARE))))
        return PFB_E_ARG;
      any = any || RS[k] >= 0;
    }
    if (!any) rowsum = nullptr;
  }
  PartsSpec PS{};
  if (parts) {
    for (int k = 0; k < n_in; ++k) {
      PS.S[k] = (int)parts[2 * k];
      PS.st[k] = parts[2 * k + 1];
      if (PS.S[k] > kMaxParts || (PS.S[k] > 1 && ins[k].dtype != PFB_F32)) return PFB_E_ARG;
    }
    if (!PS.any()) parts = nullptr;
  }
  if (n_out < 1 || n_out > kMaxOuts) return PFB_E_ARG;
  const pfb_tensor* out = &outs[0];
  for (int k = 0; k < n_out; ++k) {
    if (outs[k].dtype != PFB_F32 && outs[k].dtype != PFB_BOOL) return PFB_E_DTYPE;
    if (outs[k].rank != out->rank) return PFB_E_SHAPE;
    for (int d = 0; d < out->rank; ++d)
      if (outs[k].shape[d] != out->shape[d] || (out->shape[d] > 1 && outs[k].stride[d] != out->stride[d]))
        return PFB_E_SHAPE;
    if (out_regs[k] < 0 || out_regs[k] >= kMaxRegs) return PFB_E_ARG;
  }
  int64_t stb[kMaxIn][kMaxRank];
  const int64_t* st[kMaxFOps];
  st[0] = out->stride;
  FusedProgram P;
  P.n_in = n_in;
  P.n_steps = n_steps;
  for (int k = 0; k < n_in; ++k) {
    if (ins[k].dtype == PFB_I64) return PFB_E_DTYPE;
    if (!broadcast_strides(&ins[k], out->rank, out->shape, stb[k])) return PFB_E_SHAPE;
    st[k + 1] = stb[k];
    P.in_dtype[k] = ins[k].dtype;
  }
  for (int k = n_in; k < kMaxIn; ++k) P.in_dtype[k] = PFB_F32;
  for (int s = 0; s < n_steps; ++s) {
    for (int j = 0; j < 4; ++j) P.code[s][j] = program[4 * s + j];
    if (P.code[s][1] < 0 || P.code[s][1] >= kMaxRegs) return PFB_E_ARG;
  }
  FusedOuts fo;
  P.n_out = n_out;
  for (int k = 0; k < kMaxOuts; ++k) {
    fo.p[k] = k < n_out ? outs[k].data : nullptr;
    P.out_reg[k] = k < n_out ? out_regs[k] : 0;
    P.out_dt[k] = k < n_out ? outs[k].dtype : PFB_F32;
  }
  FLayout L = make_layout<kMaxFOps>(out->rank, out->shape, n_in + 1, st);
  int64_t n = numel(out);
  if (n == 0) return 0;
  FusedIns fi;
  for (int k = 0; k < kMaxIn; ++k) fi.p[k] = k < n_in ? ins[k].data : nullptr;
  cudaStream_t s = as_stream(stream);
  const bool small = n < (int64_t)0x7fffffff;
  const int ir = L.rank - 1;
  static const bool scalar_only = getenv_flag("PFB_FUSED_SCALAR");
  // below ~1M elements (L2-resident per-step tensors: the LSTM cell, 131k
  // elements) one element per thread: the program's latency chain runs on 4x
  // the warps (cfg4 step 2.76 -> 2.58 ms); 4 per thread (128-bit accesses)
  // where the launch is HBM-bound
  const bool v4 = !rowsum && L.shape[ir] % 4 == 0 && !scalar_only && n >= (int64_t)1 << 20;
  // per-operand feed mode; the outputs share operand 0's (all must be aligned)
  FeedModes modes = 0;
  for (int o = 0; o <= n_in; ++o) {
    bool vec = v4 && L.st[o][ir] == 1;
    if (o == 0) {
      for (int k = 0; k < n_out && vec; ++k) {
        const int64_t esz = outs[k].dtype == PFB_F32 ? 4 : 1;
        vec = (reinterpret_cast<uintptr_t>(outs[k].data) % (4 * esz)) == 0;
      }
    } else {
      const int64_t esz = ins[o - 1].dtype == PFB_F32 ? 4 : 1;
      vec = vec && (reinterpret_cast<uintptr_t>(ins[o - 1].data) % (4 * esz)) == 0;
      if (parts && PS.S[o - 1] > 1) vec = vec && PS.st[o - 1] % 4 == 0;
    }
    for (int d = 0; d < ir && vec; ++d) vec = (L.st[o][d] % 4) == 0;
    const FeedModes m = (L.st[o][ir] == 0 && o > 0) ? 1u : (vec ? 0u : 2u);
    modes |= m << (2 * o);
  }
  const int64_t ng = v4 ? n / 4 : n;
  if (rowsum) {  // F16 row-sum feeds: the specialised row kernel or nothing
    if (!fused_rows_jit_launch(P, modes, L, n, fo, fi, s, parts ? &PS : nullptr, RS))
      return PFB_E_UNSUPPORTED;
    return launch_status();
  }
  if (fused_jit_launch(P, v4 ? 4 : 1, !small, modes, L, ng, fo, fi, s, parts ? &PS : nullptr))
    return launch_status();
  if (parts) return PFB_E_UNSUPPORTED;  // partial sums: specialised kernels only
  if (v4) {
    if (small) launch_fused<4, uint32_t>(n_in, L, (uint32_t)ng, P, modes, fo, fi, s);
    else launch_fused<4, int64_t>(n_in, L, ng, P, modes, fo, fi, s);
  } else {
    if (small) launch_fused<1, uint32_t>(n_in, L, (uint32_t)ng, P, modes, fo, fi, s);
    else launch_fused<1, int64_t>(n_in, L, ng, P, modes, fo, fi, s);
  }
  return launch_status();
}

extern "C" int pfb_fused_ew(int32_t n_in, const pfb_tensor* ins, int32_t n_steps,
                            const int32_t* program, pfb_tensor* out, void* stream) {
  if (n_steps < 1 || n_steps > kMaxSteps) return PFB_E_ARG;
  const int32_t last = program[4 * (n_steps - 1) + 1];
  return fused_impl(n_in, ins, n_steps, program, 1, &last, out, stream);
}

extern "C" int pfb_fused_ew_multi(int32_t n_in, const pfb_tensor* ins, int32_t n_steps,
                                  const int32_t* program, int32_t n_out, const int32_t* out_regs,
                                  pfb_tensor* outs, void* stream) {
  return fused_impl(n_in, ins, n_steps, program, n_out, out_regs, outs, stream);
}

extern "C" int pfb_fused_ew_parts(int32_t n_in, const pfb_tensor* ins, const int64_t* parts,
                                  int32_t n_steps, const int32_t* program, int32_t n_out,
                                  const int32_t* out_regs, pfb_tensor* outs, void* stream) {
  return fused_impl(n_in, ins, n_steps, program, n_out, out_regs, outs, stream, parts);
}

extern "C" int pfb_fused_ew_rows(int32_t n_in, const pfb_tensor* ins, const int64_t* parts,
                                 const int32_t* rowsum, int32_t n_steps, const int32_t* program,
                                 int32_t n_out, const int32_t* out_regs, pfb_tensor* outs,
                                 void* stream) {
  return fused_impl(n_in, ins, n_steps, program, n_out, out_regs, outs, stream, parts, rowsum);
}

// ---------------------------------------------------------------------------
// select(mask, a, b) = mask ? a : b  (predicated control flow; numpy.where)

namespace pfb {
template <typename T, typename IdxT>
__global__ void __launch_bounds__(256) select_kernel(Layout L, IdxT n, T* out, const uint8_t* m,
                                                     const T* a, const T* b) {
  pdl_enter();
  for (IdxT i = blockIdx.x * (IdxT)blockDim.x + threadIdx.x; i < n;
       i += (IdxT)gridDim.x * blockDim.x) {
    int64_t off[4];
    offsets<IdxT, 4>(L, i, off);
    out[off[0]] = __ldg(m + off[1]) ? __ldg(a + off[2]) : __ldg(b + off[3]);
  }
}

template <typename T>
int select_run(const Layout& L, int64_t n, pfb_tensor* out, const pfb_tensor* m,
               const pfb_tensor* a, const pfb_tensor* b, cudaStream_t s) {
  const int grid = grid_for(n, 256);
  if (n < (int64_t)0x7fffffff)
    launch(select_kernel<T, uint32_t>, grid, 256, 0, s, L, (uint32_t)n, (T*)out->data,
                                                    (const uint8_t*)m->data, (const T*)a->data,
                                                    (const T*)b->data);
  else
    launch(select_kernel<T, int64_t>, grid, 256, 0, s, L, n, (T*)out->data, (const uint8_t*)m->data,
                                                   (const T*)a->data, (const T*)b->data);
  return launch_status();
}
}  // namespace pfb

extern "C" int pfb_select(const pfb_tensor* mask, const pfb_tensor* a, const pfb_tensor* b,
                          pfb_tensor* out, void* stream) {
  using namespace pfb;
  if (mask->dtype != PFB_BOOL || a->dtype != b->dtype || a->dtype != out->dtype) return PFB_E_DTYPE;
  int64_t sm[kMaxRank], sa[kMaxRank], sb[kMaxRank];
  if (!broadcast_strides(mask, out->rank, out->shape, sm) ||
      !broadcast_strides(a, out->rank, out->shape, sa) ||
      !broadcast_strides(b, out->rank, out->shape, sb))
    return PFB_E_SHAPE;
  const int64_t* st[4] = {out->stride, sm, sa, sb};
  Layout L = make_layout(out->rank, out->shape, 4, st);
  int64_t n = numel(out);
  if (n == 0) return 0;
  cudaStream_t s = as_stream(stream);
  switch (a->dtype) {
    case PFB_F32: return select_run<float>(L, n, out, mask, a, b, s);
    case PFB_I64: return select_run<int64_t>(L, n, out, mask, a, b, s);
    default: return select_run<uint8_t>(L, n, out, mask, a, b, s);
  }
}

// ---------------------------------------------------------------------------
// concat of up to kMaxCat same-dtype inputs along one axis in one launch
// (reference tensor.concat, tensor.py:383-393): blockIdx.y picks the input,
// threads stride over its elements; each input may be any strided view.

namespace pfb {
constexpr int kMaxCat = 24;
struct CatDesc {
  int rank, ax, n;
  int64_t shape[kMaxRank];      // common shape (axis extent per input below)
  int64_t ost[kMaxRank];        // output strides
  const void* x[kMaxCat];
  int64_t ext[kMaxCat], off[kMaxCat];
  int64_t xst[kMaxCat][kMaxRank];
};

template <typename T>
__global__ void __launch_bounds__(256) concat_kernel(CatDesc d, T* out) {
  pdl_enter();
  const int j = blockIdx.y;
  int64_t numel = 1;
  for (int i = 0; i < d.rank; ++i) numel *= (i == d.ax ? d.ext[j] : d.shape[i]);
  const T* x = reinterpret_cast<const T*>(d.x[j]);
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < numel;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = lin, xo = 0, oo = d.off[j] * d.ost[d.ax];
    for (int i = d.rank - 1; i >= 0; --i) {
      const int64_t e = (i == d.ax ? d.ext[j] : d.shape[i]);
      const int64_t q = r / e, c = r - q * e;
      xo += c * d.xst[j][i];
      oo += c * d.ost[i];
      r = q;
    }
    out[oo] = __ldg(x + xo);
  }
}
// Concat of many width-1 inputs along a contiguous innermost axis (cfg4's F2
// operands: 64 [n,1024,1] columns -> [n,1024,64]).  The generic kernel walks
// each input and writes one float per 256-byte output row; here a 32x32 tile
// is transposed through shared memory: every input column is read as 128
// contiguous bytes and every output row segment written as 128 bytes.
constexpr int kThinCat = 128;
struct ThinCat {
  int n;
  int64_t R, R1, ost_row, off;  // R rows = R0 x R1 (outer x inner row dims)
  const void* x[kThinCat];
  int64_t rs0[kThinCat], rs1[kThinCat];  // per input: outer / inner row strides
};

constexpr int kThinRows = 128;  // rows per block (4 x 32: 16 loads in flight per thread)

template <typename T>
__global__ void __launch_bounds__(256) concat_thin_kernel(ThinCat d, T* out) {
  pdl_enter();
  __shared__ T tile[32][kThinRows + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * kThinRows;
  const int c0 = blockIdx.y * 32;
  T v[4][kThinRows / 32];
#pragma unroll
  for (int q = 0; q < kThinRows / 32; ++q) {
    const int64_t r = r0 + q * 32 + tx;
    const int64_t ro = r / d.R1, ri = r - ro * d.R1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = c0 + ty + 8 * k;
      v[k][q] = (c < d.n && r < d.R)
                    ? __ldg(reinterpret_cast<const T*>(d.x[c]) + ro * d.rs0[c] + ri * d.rs1[c])
                    : T(0);
    }
  }
#pragma unroll
  for (int q = 0; q < kThinRows / 32; ++q)
#pragma unroll
    for (int k = 0; k < 4; ++k) tile[ty + 8 * k][q * 32 + tx] = v[k][q];
  __syncthreads();
  const int c = c0 + tx;
#pragma unroll 4
  for (int i = ty; i < kThinRows; i += 8) {
    const int64_t rr = r0 + i;
    if (c < d.n && rr < d.R) out[rr * d.ost_row + d.off + c] = tile[tx][i];
  }
}

// Concat of dense inputs into a dense output: each input is a [rows, inner_j]
// block copied into columns [off_j, off_j + inner_j) of the [rows, inner]
// output -- 16-byte loads/stores when every width and offset allows it
// (the generic kernel decodes every element's coordinates instead).
struct RowCat {
  int n;
  int64_t rows, inner;
  const void* x[kMaxCat];
  int64_t w[kMaxCat], off[kMaxCat];
  int64_t rs[kMaxCat];  // input row stride (elements): w for a dense input
};

template <typename T, int V>
__global__ void __launch_bounds__(256) concat_rows_kernel(RowCat d, T* out) {
  pdl_enter();
  const int j = blockIdx.y;
  const int64_t wv = d.w[j] / V, total = d.rows * wv;
  const T* x = reinterpret_cast<const T*>(d.x[j]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / wv, c = i - r * wv;
    if constexpr (V == 4 && sizeof(T) == 4) {
      *reinterpret_cast<float4*>(out + r * d.inner + d.off[j] + 4 * c) =
          __ldg(reinterpret_cast<const float4*>(x + r * d.rs[j] + 4 * c));
    } else {
      out[r * d.inner + d.off[j] + c] = __ldg(x + r * d.rs[j] + c);
    }
  }
}

static bool concat_rows(int32_t n, const pfb_tensor* xs, int32_t axis, pfb_tensor* out,
                        cudaStream_t s) {
  if (!is_dense(out) || n > kMaxCat) return false;
  RowCat d;
  d.n = n;
  d.rows = 1;
  for (int i = 0; i < axis; ++i) d.rows *= out->shape[i];
  d.inner = 1;
  for (int i = axis; i < out->rank; ++i) d.inner *= out->shape[i];
  int64_t post = 1;
  for (int i = axis + 1; i < out->rank; ++i) post *= out->shape[i];
  bool v4 = out->dtype == PFB_F32 && (reinterpret_cast<uintptr_t>(out->data) & 15) == 0 &&
            d.inner % 4 == 0;
  int64_t off = 0, most = 0;
  for (int j = 0; j < n; ++j) {
    const pfb_tensor* x = &xs[j];
    if (x->dtype != out->dtype || x->rank != out->rank) return false;
    for (int i = 0; i < out->rank; ++i)
      if (i != axis && x->shape[i] != out->shape[i]) return false;
    // the input as [rows, w] rows: dims axis.. contiguous, dims ..axis one
    // stride (a dense input, or a row-strided slice such as one time step
    // of a [n, T, d] tensor)
    int64_t expect = 1;
    for (int i = out->rank - 1; i >= axis; --i) {
      if (x->shape[i] != 1 && x->stride[i] != expect) return false;
      expect *= x->shape[i];
    }
    int64_t rs = -1, next = -1;
    for (int i = axis - 1; i >= 0; --i) {
      if (x->shape[i] == 1) continue;
      if (rs < 0) { rs = x->stride[i]; next = rs * x->shape[i]; continue; }
      if (x->stride[i] != next) return false;
      next *= x->shape[i];
    }
    d.x[j] = x->data;
    d.w[j] = x->shape[axis] * post;
    d.rs[j] = rs < 0 ? d.w[j] : rs;
    d.off[j] = off;
    off += d.w[j];
    most = std::max(most, d.rows * d.w[j]);
    v4 = v4 && d.w[j] % 4 == 0 && d.off[j] % 4 == 0 && d.rs[j] % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(x->data) & 15) == 0;
  }
  if (off != d.inner || most == 0) return off == d.inner;
  const int gx = grid_for(v4 ? most / 4 : most, 256, 4);
  dim3 grid((unsigned)gx, (unsigned)n);
  if (v4) {
    launch(concat_rows_kernel<float, 4>, grid, 256, 0, s, d, (float*)out->data);
  } else {
    switch (out->dtype) {
      case PFB_F32: launch(concat_rows_kernel<float, 1>, grid, 256, 0, s, d, (float*)out->data); break;
      case PFB_I64: launch(concat_rows_kernel<int64_t, 1>, grid, 256, 0, s, d, (int64_t*)out->data); break;
      default: launch(concat_rows_kernel<uint8_t, 1>, grid, 256, 0, s, d, (uint8_t*)out->data); break;
    }
  }
  return true;
}

// leading dims [0, rank-1) of a view collapsed into one stride, or -1
static int64_t collapse_rows(const pfb_tensor* t, int rank) {
  int64_t st = -1, expect = -1;
  for (int i = rank - 2; i >= 0; --i) {
    if (t->shape[i] == 1) continue;
    if (st < 0) { st = t->stride[i]; expect = st * t->shape[i]; continue; }
    if (t->stride[i] != expect) return -1;
    expect *= t->shape[i];
  }
  return st < 0 ? 0 : st;
}

// rows of a [.., R1, 1] view as (outer, inner) strides: dims [0, rank-2)
// collapsed into one outer stride, dim rank-2 the inner one; false when the
// outer dims do not collapse
static bool rows2(const pfb_tensor* t, int rank, int64_t* s0, int64_t* s1) {
  *s1 = t->shape[rank - 2] == 1 ? 0 : t->stride[rank - 2];
  int64_t st = -1, expect = -1;
  for (int i = rank - 3; i >= 0; --i) {
    if (t->shape[i] == 1) continue;
    if (st < 0) { st = t->stride[i]; expect = st * t->shape[i]; continue; }
    if (t->stride[i] != expect) return false;
    expect *= t->shape[i];
  }
  *s0 = st < 0 ? 0 : st;
  return true;
}

static bool concat_thin(int32_t n, const pfb_tensor* xs, int32_t axis, pfb_tensor* out,
                        cudaStream_t s) {
  const int rank = out->rank;
  if (axis != rank - 1 || rank < 2 || out->stride[axis] != 1 || n < 8) return false;
  if (out->shape[axis] != n) return false;
  ThinCat d;
  d.R = 1;
  for (int i = 0; i < rank - 1; ++i) d.R *= out->shape[i];
  d.R1 = out->shape[rank - 2];
  d.ost_row = collapse_rows(out, rank);
  if (d.ost_row < 0 || d.R == 0 || d.R1 == 0) return false;
  for (int j = 0; j < n; ++j) {
    const pfb_tensor* x = &xs[j];
    if (x->rank != rank || x->shape[axis] != 1 || x->dtype != out->dtype) return false;
    for (int i = 0; i < rank - 1; ++i)
      if (x->shape[i] != out->shape[i]) return false;
    int64_t a, b;
    if (!rows2(x, rank, &a, &b)) return false;
  }
  for (int base = 0; base < n; base += kThinCat) {
    d.n = std::min(kThinCat, n - base);
    d.off = base;
    for (int j = 0; j < d.n; ++j) {
      d.x[j] = xs[base + j].data;
      rows2(&xs[base + j], rank, &d.rs0[j], &d.rs1[j]);
    }
    dim3 grid((unsigned)((d.R + kThinRows - 1) / kThinRows), (unsigned)((d.n + 31) / 32));
    switch (out->dtype) {
      case PFB_F32: launch(concat_thin_kernel<float>, grid, 256, 0, s, d, (float*)out->data); break;
      case PFB_I64: launch(concat_thin_kernel<int64_t>, grid, 256, 0, s, d, (int64_t*)out->data); break;
      default: launch(concat_thin_kernel<uint8_t>, grid, 256, 0, s, d, (uint8_t*)out->data); break;
    }
  }
  return true;
}
}  // namespace pfb

extern "C" int pfb_concat(int32_t n, const pfb_tensor* xs, int32_t axis, pfb_tensor* out,
                          void* stream) {
  using namespace pfb;
  if (n < 1) return PFB_E_ARG;
  const int rank = out->rank;
  if (axis < 0 || axis >= rank) return PFB_E_ARG;
  cudaStream_t s = as_stream(stream);
  if (concat_thin(n, xs, axis, out, s)) return launch_status();
  if (concat_rows(n, xs, axis, out, s)) return launch_status();
  int64_t off = 0;
  for (int base = 0; base < n; base += kMaxCat) {
    CatDesc d;
    d.rank = rank;
    d.ax = axis;
    d.n = std::min(kMaxCat, n - base);
    int64_t maxel = 0;
    for (int i = 0; i < rank; ++i) {
      d.shape[i] = out->shape[i];
      d.ost[i] = out->stride[i];
    }
    for (int j = 0; j < d.n; ++j) {
      const pfb_tensor* x = &xs[base + j];
      if (x->dtype != out->dtype) return PFB_E_DTYPE;
      if (x->rank != rank) return PFB_E_RANK;
      for (int i = 0; i < rank; ++i)
        if (i != axis && x->shape[i] != out->shape[i]) return PFB_E_SHAPE;
      d.x[j] = x->data;
      d.ext[j] = x->shape[axis];
      d.off[j] = off;
      off += x->shape[axis];
      for (int i = 0; i < rank; ++i) d.xst[j][i] = x->stride[i];
      maxel = std::max(maxel, numel(x));
    }
    if (off > out->shape[axis]) return PFB_E_SHAPE;
    if (maxel == 0) continue;
    dim3 grid((unsigned)grid_for(maxel, 256, 4), (unsigned)d.n);
    switch (out->dtype) {
      case PFB_F32: launch(concat_kernel<float>, grid, 256, 0, s, d, (float*)out->data); break;
      case PFB_I64: launch(concat_kernel<int64_t>, grid, 256, 0, s, d, (int64_t*)out->data); break;
      default: launch(concat_kernel<uint8_t>, grid, 256, 0, s, d, (uint8_t*)out->data); break;
    }
  }
  if (off != out->shape[axis]) return PFB_E_SHAPE;
  return launch_status();
}
