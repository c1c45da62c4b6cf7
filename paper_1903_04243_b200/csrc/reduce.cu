// reduce_sum over an axis set (reference tensor.py:267-283).
//
// The input (any strides) is split into kept dims K and reduced dims R, each
// collapsed independently.  Two schedules, both deterministic (fixed
// association order, no float atomics):
//   inner  -- the unit-stride dim is reduced: a warp (small R) or a block
//             (large R, optionally split across CTAs) per output, lanes
//             striding along R -> coalesced, warp-shuffle + smem tree;
//   outer  -- the unit-stride dim is kept: one thread per output (coalesced
//             across the warp), looping over R with Kahan compensation,
//             R split across CTAs (blockIdx.y) when there are too few outputs.
// Split schedules write per-split partials to the workspace and a second
// pass adds them in split order.  fp32 with compensated / tree summation
// keeps ~1 ulp-scale error, well inside the rtol 1e-4 bar.
#include "common.cuh"
#include <algorithm>

namespace pfb {

struct RedDesc {
  int kr, rr;
  int64_t kshape[kMaxRank], kst[kMaxRank], kst_y[kMaxRank];
  int64_t rshape[kMaxRank], rst[kMaxRank], rst_y[kMaxRank];
};

// offsets of one (kept or reduced) index for x and y at once
__device__ __forceinline__ void decode2(int rank, const int64_t* shape, const int64_t* st,
                                        const int64_t* sty, int64_t lin, int64_t* ox,
                                        int64_t* oy) {
  if (rank == 1) { *ox = lin * st[0]; *oy = lin * sty[0]; return; }
  int64_t a = 0, b = 0;
  for (int d = rank - 1; d >= 0; --d) {
    int64_t q = lin / shape[d];
    int64_t c = lin - q * shape[d];
    a += c * st[d];
    b += c * sty[d];
    lin = q;
  }
  *ox = a;
  *oy = b;
}

__device__ __forceinline__ int64_t decode(int rank, const int64_t* shape, const int64_t* st,
                                          int64_t lin) {
  if (rank == 1) return lin * st[0];
  int64_t off = 0;
  for (int d = rank - 1; d >= 0; --d) {
    int64_t q = lin / shape[d];
    off += (lin - q * shape[d]) * st[d];
    lin = q;
  }
  return off;
}

template <typename T>
struct Acc {  // Kahan-compensated for float, exact wraparound for int64
  T s = 0, c = 0;
  __device__ __forceinline__ void add(T v) {
    if constexpr (std::is_same<T, float>::value) {
      T y = v - c;
      T t = s + y;
      c = (t - s) - y;
      s = t;
    } else {
      s = (T)((uint64_t)s + (uint64_t)v);
    }
  }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    if constexpr (std::is_same<T, float>::value) v += __shfl_xor_sync(0xffffffffu, v, o);
    else v = (T)((uint64_t)v + (uint64_t)__shfl_xor_sync(0xffffffffu, (long long)v, o));
  }
  return v;
}

// x[i] (PROD: x[i] * y[i])
template <typename T, bool PROD>
__device__ __forceinline__ T elem(const RedDesc& D, const T* x, const T* y, int64_t kx,
                                  int64_t ky, int64_t r) {
  if (!PROD) return x[kx + decode(D.rr, D.rshape, D.rst, r)];
  int64_t ox, oy;
  decode2(D.rr, D.rshape, D.rst, D.rst_y, r, &ox, &oy);
  return x[kx + ox] * y[ky + oy];
}

// one warp per output; R small
template <typename T, bool PROD>
__global__ void __launch_bounds__(256) reduce_inner_warp(RedDesc D, int64_t K, int64_t R,
                                                         const T* x, const T* y, T* out) {
  pdl_enter();
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t k = blockIdx.x * 8ll + warp; k < K; k += gridDim.x * 8ll) {
    int64_t base, basey;
    decode2(D.kr, D.kshape, D.kst, D.kst_y, k, &base, &basey);
    Acc<T> acc;
    if (D.rr == 1) {  // single collapsed reduced dim: no index decode per element
      const T* p = x + base;
      const int64_t s = D.rst[0];
      if constexpr (std::is_same<T, float>::value) {
        // contiguous float row: 16-byte loads, 4 independent compensated sums
        const T* q = PROD ? y + basey : nullptr;
        const bool vec = s == 1 && (reinterpret_cast<uintptr_t>(p) & 15) == 0 &&
                         (!PROD || (D.rst_y[0] == 1 && (reinterpret_cast<uintptr_t>(q) & 15) == 0));
        if (vec) {
          Acc<T> a4[4];
          const int64_t R4 = R / 4;
          for (int64_t r = lane; r < R4; r += 32) {
            float4 v = __ldg(reinterpret_cast<const float4*>(p) + r);
            if (PROD) {
              const float4 w = __ldg(reinterpret_cast<const float4*>(q) + r);
              v.x *= w.x; v.y *= w.y; v.z *= w.z; v.w *= w.w;
            }
            a4[0].add(v.x); a4[1].add(v.y); a4[2].add(v.z); a4[3].add(v.w);
          }
          for (int64_t r = 4 * R4 + lane; r < R; r += 32)
            a4[0].add(PROD ? __ldg(p + r) * __ldg(q + r) : __ldg(p + r));
          acc.add(a4[0].s); acc.add(a4[1].s); acc.add(a4[2].s); acc.add(a4[3].s);
          T v = warp_sum(acc.s);
          if (lane == 0) out[k] = v;
          continue;
        }
      }
      if (PROD) {
        const T* q = y + basey;
        const int64_t sy = D.rst_y[0];
        for (int64_t r = lane; r < R; r += 32) acc.add(__ldg(p + r * s) * __ldg(q + r * sy));
      } else {
        for (int64_t r = lane; r < R; r += 32) acc.add(__ldg(p + r * s));
      }
    } else {
      for (int64_t r = lane; r < R; r += 32) acc.add(elem<T, PROD>(D, x, y, base, basey, r));
    }
    T v = warp_sum(acc.s);
    if (lane == 0) out[k] = v;
  }
}

// short contiguous float rows (R <= 128, R % 4 == 0, one reduced dim of
// unit stride): LPR = R/4 lanes (a power of two) per row, 32/LPR rows per
// warp, one 16-byte load per lane; 4 row groups are loaded before any is
// reduced, so a warp keeps 4 loads in flight instead of one row's worth
template <int LPR>
__global__ void __launch_bounds__(256) reduce_inner_short(RedDesc D, int64_t K, int R4,
                                                          const float* __restrict__ x,
                                                          float* __restrict__ out) {
  pdl_enter();
  constexpr int RPW = 32 / LPR;  // rows per warp pass
  const int lane = threadIdx.x & 31, sub = lane % LPR, rw = lane / LPR;
  const int64_t warps = (int64_t)gridDim.x * 8;
  const int64_t w0 = blockIdx.x * 8ll + (threadIdx.x >> 5);
  for (int64_t k0 = w0 * RPW * 4; k0 < K; k0 += warps * RPW * 4) {
    float4 v[4];
    int64_t kk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      kk[u] = k0 + u * RPW + rw;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kk[u] < K && sub < R4)
        v[u] = __ldg(reinterpret_cast<const float4*>(x + decode(D.kr, D.kshape, D.kst, kk[u])) + sub);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float t = (v[u].x + v[u].y) + (v[u].z + v[u].w);
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (sub == 0 && kk[u] < K) out[kk[u]] = t;
    }
  }
}

// block per (output, split); partial -> out[k] (nsplit==1) or ws[k*nsplit+split]
template <typename T, bool PROD>
__global__ void __launch_bounds__(256) reduce_inner_block(RedDesc D, int64_t K, int64_t R,
                                                          int nsplit, const T* x, const T* y,
                                                          T* dst) {
  pdl_enter();
  __shared__ T red[8];
  int64_t k = blockIdx.x / nsplit;
  int split = blockIdx.x % nsplit;
  int64_t chunk = (R + nsplit - 1) / nsplit;
  int64_t r0 = split * chunk, r1 = min(R, r0 + chunk);
  int64_t base, basey;
  decode2(D.kr, D.kshape, D.kst, D.kst_y, k, &base, &basey);
  Acc<T> acc;
  if (!PROD && D.rr == 1 && D.rst[0] == 1) {
    const T* p = x + base;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) acc.add(__ldg(p + r));
  } else {
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x)
      acc.add(elem<T, PROD>(D, x, y, base, basey, r));
  }
  T v = warp_sum(acc.s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    T w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : (T)0;
    w = warp_sum(w);
    if (threadIdx.x == 0) dst[nsplit == 1 ? k : k * nsplit + split] = w;
  }
}

// thread per output, loop over an R chunk (blockIdx.y = split)
template <typename T, bool PROD>
__global__ void __launch_bounds__(256) reduce_outer(RedDesc D, int64_t K, int64_t R, int nsplit,
                                                    const T* x, const T* y, T* dst) {
  pdl_enter();
  int split = blockIdx.y;
  int64_t chunk = (R + nsplit - 1) / nsplit;
  int64_t r0 = split * chunk, r1 = min(R, r0 + chunk);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t base, basey;
    decode2(D.kr, D.kshape, D.kst, D.kst_y, k, &base, &basey);
    Acc<T> acc;
    if (D.rr == 1) {
      const T* p = x + base;
      const int64_t s = D.rst[0];
      if (PROD) {
        const T* q = y + basey;
        const int64_t sy = D.rst_y[0];
        for (int64_t r = r0; r < r1; ++r) acc.add(__ldg(p + r * s) * __ldg(q + r * sy));
      } else {
        for (int64_t r = r0; r < r1; ++r) acc.add(__ldg(p + r * s));
      }
    } else {
      for (int64_t r = r0; r < r1; ++r) acc.add(elem<T, PROD>(D, x, y, base, basey, r));
    }
    dst[nsplit == 1 ? k : split * K + k] = acc.s;
  }
}

// Outer reduction over a contiguous kept dim (fp32): a thread owns 4 adjacent
// outputs (one 16-byte load per row) and 2 rows per trip, so each thread keeps
// 32 bytes in flight per trip; R is split over blockIdx.y into partials
// (ws[split*K + k]) added in split order by combine_partials.
template <bool PROD>
__global__ void __launch_bounds__(256) reduce_outer_vec(int64_t K4, int64_t R, int nsplit,
                                                        const float* x, int64_t sx,
                                                        const float* y, int64_t sy,
                                                        float* dst) {
  pdl_enter();
  const int split = blockIdx.y;
  const int64_t chunk = (R + nsplit - 1) / nsplit;
  const int64_t r0 = split * chunk, r1 = min(R, r0 + chunk);
  const int64_t k4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k4 >= K4) return;
  Acc<float> a[2][4];
  auto row = [&](int64_t r) {
    float4 v = __ldg(reinterpret_cast<const float4*>(x + r * sx) + k4);
    if (PROD) {
      const float4 w = __ldg(reinterpret_cast<const float4*>(y + r * sy) + k4);
      v.x *= w.x; v.y *= w.y; v.z *= w.z; v.w *= w.w;
    }
    return v;
  };
  int64_t r = r0;
  for (; r + 1 < r1; r += 2) {
    const float4 v0 = row(r), v1 = row(r + 1);
    a[0][0].add(v0.x); a[0][1].add(v0.y); a[0][2].add(v0.z); a[0][3].add(v0.w);
    a[1][0].add(v1.x); a[1][1].add(v1.y); a[1][2].add(v1.z); a[1][3].add(v1.w);
  }
  if (r < r1) {
    const float4 v0 = row(r);
    a[0][0].add(v0.x); a[0][1].add(v0.y); a[0][2].add(v0.z); a[0][3].add(v0.w);
  }
  float4 o;
  a[0][0].add(a[1][0].s); a[0][1].add(a[1][1].s); a[0][2].add(a[1][2].s); a[0][3].add(a[1][3].s);
  o.x = a[0][0].s; o.y = a[0][1].s; o.z = a[0][2].s; o.w = a[0][3].s;
  reinterpret_cast<float4*>(dst + (nsplit == 1 ? 0 : split * K4 * 4))[k4] = o;
}

// Outer reduction in one launch for moderate R: a block owns 32 outputs
// (lanes) and splits R over its 8 warps; the 8 partial sums are combined in
// warp order through shared memory (deterministic, no second pass).
template <typename T, bool PROD>
__global__ void __launch_bounds__(256) reduce_outer_tile(RedDesc D, int64_t K, int64_t R,
                                                         const T* x, const T* y, T* dst) {
  pdl_enter();
  __shared__ T part[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t k = (int64_t)blockIdx.x * 32 + lane;
  const int64_t chunk = (R + 7) / 8;
  const int64_t r0 = grp * chunk, r1 = min(R, r0 + chunk);
  Acc<T> acc;
  if (k < K) {
    int64_t base, basey;
    decode2(D.kr, D.kshape, D.kst, D.kst_y, k, &base, &basey);
    if (D.rr == 1) {
      const T* p = x + base;
      const int64_t st = D.rst[0];
      if (PROD) {
        const T* q = y + basey;
        const int64_t sy = D.rst_y[0];
        for (int64_t r = r0; r < r1; ++r) acc.add(__ldg(p + r * st) * __ldg(q + r * sy));
      } else {
        for (int64_t r = r0; r < r1; ++r) acc.add(__ldg(p + r * st));
      }
    } else {
      for (int64_t r = r0; r < r1; ++r) acc.add(elem<T, PROD>(D, x, y, base, basey, r));
    }
  }
  part[grp][lane] = acc.s;
  __syncthreads();
  if (grp == 0 && k < K) {
    Acc<T> tot;
#pragma unroll
    for (int g = 0; g < 8; ++g) tot.add(part[g][lane]);
    dst[k] = tot.s;
  }
}

template <typename T>
__global__ void sum_partials(int64_t K, int nsplit, bool k_major, const T* ws, T* out) {
  pdl_enter();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K;
       k += (int64_t)gridDim.x * blockDim.x) {
    Acc<T> acc;
    for (int s = 0; s < nsplit; ++s) acc.add(k_major ? ws[k * nsplit + s] : ws[s * K + k]);
    out[k] = acc.s;
  }
}

template <typename T>
__global__ void fill_zero(int64_t n, T* out) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)0;
}

// partials [ns, K] -> out[K]: 8 warps per 32 outputs, fixed combine order
template <typename T>
static void combine_partials(int64_t K, int ns, const T* ws, T* o, cudaStream_t s) {
  RedDesc P{};
  P.kr = 1; P.kshape[0] = K; P.kst[0] = 1;
  P.rr = 1; P.rshape[0] = ns; P.rst[0] = K;
  launch(reduce_outer_tile<T, false>, (unsigned)((K + 31) / 32), 256, 0, s, P, K, (int64_t)ns, ws,
         (const T*)nullptr, o);
}

static int collapse(int n, int64_t* shape, int64_t* st, int64_t* sty) {
  int w = 0;
  for (int d = 0; d < n; ++d) {
    if (shape[d] == 1) continue;
    if (w > 0 && st[w - 1] == st[d] * shape[d] && sty[w - 1] == sty[d] * shape[d]) {
      shape[w - 1] *= shape[d];
      st[w - 1] = st[d];
      sty[w - 1] = sty[d];
      continue;
    }
    shape[w] = shape[d];
    st[w] = st[d];
    sty[w] = sty[d];
    ++w;
  }
  if (w == 0) { shape[0] = 1; st[0] = 0; sty[0] = 0; w = 1; }
  return w;
}

template <typename T, bool PROD>
int reduce_run(const pfb_tensor* x, const int64_t* ystride, const T* yp, uint32_t mask,
               pfb_tensor* out, void* ws, int64_t ws_bytes, cudaStream_t s) {
  RedDesc D;
  int nk = 0, nr = 0;
  int64_t K = 1, R = 1;
  for (int d = 0; d < x->rank; ++d) {
    const int64_t sy = PROD ? ystride[d] : 0;
    if (mask & (1u << d)) {
      D.rshape[nr] = x->shape[d]; D.rst[nr] = x->stride[d]; D.rst_y[nr] = sy; ++nr;
      R *= x->shape[d];
    } else {
      D.kshape[nk] = x->shape[d]; D.kst[nk] = x->stride[d]; D.kst_y[nk] = sy; ++nk;
      K *= x->shape[d];
    }
  }
  if (numel(out) != K) return PFB_E_SHAPE;
  if (!is_dense(out)) return PFB_E_UNSUPPORTED;
  if (K == 0) return 0;
  T* o = (T*)out->data;
  if (R == 0) {
    launch(fill_zero<T>, grid_for(K, 256), 256, 0, s, K, o);
    return launch_status();
  }
  int64_t kinner = 0, rinner = 0;  // smallest non-trivial stride on each side
  for (int d = 0; d < nk; ++d) if (D.kshape[d] > 1 && (kinner == 0 || llabs(D.kst[d]) < kinner)) kinner = llabs(D.kst[d]);
  for (int d = 0; d < nr; ++d) if (D.rshape[d] > 1 && (rinner == 0 || llabs(D.rst[d]) < rinner)) rinner = llabs(D.rst[d]);
  D.kr = collapse(nk, D.kshape, D.kst, D.kst_y);
  D.rr = collapse(nr, D.rshape, D.rst, D.rst_y);
  const T* xp = (const T*)x->data;
  bool inner = (K == 1) || (rinner != 0 && (kinner == 0 || rinner < kinner));
  if (inner) {
    if constexpr (std::is_same<T, float>::value && !PROD) {
      // short rows: several rows per warp (cfg4's bias gradient: R = T = 64)
      bool aligned = D.rr == 1 && D.rst[0] == 1 && R % 4 == 0 && R <= 128 && K > 1 &&
                     (reinterpret_cast<uintptr_t>(xp) & 15) == 0;
      for (int d = 0; d < D.kr && aligned; ++d) aligned = D.kshape[d] == 1 || D.kst[d] % 4 == 0;
      if (aligned) {
        const int R4 = (int)(R / 4);
        const int lpr = R4 <= 4 ? 4 : (R4 <= 8 ? 8 : (R4 <= 16 ? 16 : 32));
        const int64_t per_block = 8 * (32 / lpr) * 4;  // rows per block per pass
        const unsigned grid =
            (unsigned)std::min<int64_t>((K + per_block - 1) / per_block, (int64_t)kNumSMs * 32);
        if (lpr == 4) launch(reduce_inner_short<4>, grid, 256, 0, s, D, K, R4, xp, o);
        else if (lpr == 8) launch(reduce_inner_short<8>, grid, 256, 0, s, D, K, R4, xp, o);
        else if (lpr == 16) launch(reduce_inner_short<16>, grid, 256, 0, s, D, K, R4, xp, o);
        else launch(reduce_inner_short<32>, grid, 256, 0, s, D, K, R4, xp, o);
        return launch_status();
      }
    }
    if (R <= 16384 && K > 1) {
      launch(reduce_inner_warp<T, PROD>, grid_for(K, 8, 64), 256, 0, s, D, K, R, xp, yp, o);
      return launch_status();
    }
    int nsplit = 1;
    if (K < 2 * kNumSMs && R >= (1 << 16)) {
      nsplit = (int)std::min<int64_t>((4 * kNumSMs + K - 1) / K, R / 8192 + 1);
      if ((int64_t)nsplit * K * (int64_t)sizeof(T) > ws_bytes || ws == nullptr) nsplit = 1;
    }
    launch(reduce_inner_block<T, PROD>, (unsigned)(K * nsplit), 256, 0, s, D, K, R, nsplit, xp, yp,
                                                                  nsplit == 1 ? o : (T*)ws);
    if (nsplit > 1) launch(sum_partials<T>, grid_for(K, 256), 256, 0, s, K, nsplit, true, (const T*)ws, o);
    return launch_status();
  }
  if (K <= 8192 && R <= 512 && R >= 16) {
    // few outputs, moderate R: single-launch tile reduction
    launch(reduce_outer_tile<T, PROD>, (unsigned)((K + 31) / 32), 256, 0, s, D, K, R, xp, yp, o);
    return launch_status();
  }
  if constexpr (std::is_same<T, float>::value) {
    const float* yq = PROD ? (const float*)yp : nullptr;
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (D.kr == 1 && D.rr == 1 && D.kst[0] == 1 && K % 4 == 0 && D.rst[0] % 4 == 0 && al16(xp) &&
        al16(o) && (!PROD || (D.kst_y[0] == 1 && D.rst_y[0] % 4 == 0 && al16(yq))) && R >= 64) {
      const int64_t K4 = K / 4;
      const int gxv = (int)((K4 + 255) / 256);
      int ns = (int)std::min<int64_t>(R / 16, (8ll * kNumSMs) / gxv + 1);
      ns = max(1, min(ns, 1024));
      if ((int64_t)ns * K * (int64_t)sizeof(T) > ws_bytes || ws == nullptr) ns = 1;
      dim3 grid(gxv, ns);
      launch(reduce_outer_vec<PROD>, grid, 256, 0, s, K4, R, ns, xp, D.rst[0], yq,
             PROD ? D.rst_y[0] : (int64_t)0, ns == 1 ? o : (float*)ws);
      if (ns > 1) combine_partials<T>(K, ns, (const T*)ws, o, s);
      return launch_status();
    }
  }
  int gx = grid_for(K, 256, 8);
  int nsplit = 1;
  if ((int64_t)gx * 256 < 4ll * kNumSMs * 256 && R >= 64) {
    nsplit = (int)std::min<int64_t>(R / 32, (4ll * kNumSMs * 256) / ((int64_t)gx * 256) + 1);
    nsplit = max(1, min(nsplit, 1024));
    if ((int64_t)nsplit * K * (int64_t)sizeof(T) > ws_bytes || ws == nullptr) nsplit = 1;
  }
  dim3 grid(gx, nsplit);
  launch(reduce_outer<T, PROD>, grid, 256, 0, s, D, K, R, nsplit, xp, yp, nsplit == 1 ? o : (T*)ws);
  if (nsplit > 1) combine_partials<T>(K, nsplit, (const T*)ws, o, s);
  return launch_status();
}

}  // namespace pfb

extern "C" int pfb_reduce_sum(const pfb_tensor* x, uint32_t axes_mask, pfb_tensor* out, void* ws,
                              int64_t ws_bytes, void* stream) {
  using namespace pfb;
  if (x->dtype != out->dtype) return PFB_E_DTYPE;
  cudaStream_t s = as_stream(stream);
  if (x->dtype == PFB_F32)
    return reduce_run<float, false>(x, nullptr, nullptr, axes_mask, out, ws, ws_bytes, s);
  if (x->dtype == PFB_I64)
    return reduce_run<int64_t, false>(x, nullptr, nullptr, axes_mask, out, ws, ws_bytes, s);
  return PFB_E_DTYPE;  // bools are cast to i64 by the executor first
}

// sum over axes of x * y (y broadcast to x's shape): fused square / scaled
// reductions (passes.py F4) -- the product is never written to HBM.
extern "C" int pfb_reduce_dot(const pfb_tensor* x, const pfb_tensor* y, uint32_t axes_mask,
                              pfb_tensor* out, void* ws, int64_t ws_bytes, void* stream) {
  using namespace pfb;
  if (x->dtype != PFB_F32 || y->dtype != PFB_F32 || out->dtype != PFB_F32) return PFB_E_DTYPE;
  int64_t sy[kMaxRank];
  if (!broadcast_strides(y, x->rank, x->shape, sy)) return PFB_E_SHAPE;
  return reduce_run<float, true>(x, sy, (const float*)y->data, axes_mask, out, ws, ws_bytes,
                                 as_stream(stream));
}

// ---------------------------------------------------------------------------
// Several row-dots in one launch (passes.fuse_row_dots): for pair j,
// out_j[i] = sum_k x_j[i, k] * y_j[i, k] over the dense trailing part of
// rank-2 views [rows, inner_j] (row stride arbitrary, unit inner stride).
// The per-example gradient norms of a network (one |g|^2 per parameter
// block) are independent reductions of the same length-n leading dim; one
// launch replaces one per block.  One CTA per (row, pair); Kahan per thread,
// warp-shuffle + smem tree across the CTA: deterministic.

namespace pfb {
constexpr int kMaxDots = 8;
struct RowDots {
  int n;
  int64_t rows;
  const float* x[kMaxDots];
  const float* y[kMaxDots];
  int64_t inner[kMaxDots], sx[kMaxDots], sy[kMaxDots];
  float* out[kMaxDots];
  int64_t so[kMaxDots];
  int vec[kMaxDots];  // x and y rows 16-byte aligned with inner % 4 == 0
};

__global__ void __launch_bounds__(256) row_dots_kernel(RowDots d) {
  pdl_enter();
  const int j = blockIdx.y;
  const int64_t i = blockIdx.x;
  const float* x = d.x[j] + i * d.sx[j];
  const float* y = d.y[j] + i * d.sy[j];
  const int64_t inner = d.inner[j];
  Acc<float> acc;
  if (d.vec[j]) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const float4* y4 = reinterpret_cast<const float4*>(y);
    for (int64_t k = threadIdx.x; k < inner / 4; k += blockDim.x) {
      const float4 a = __ldg(x4 + k), b = __ldg(y4 + k);
      acc.add(a.x * b.x + a.y * b.y + (a.z * b.z + a.w * b.w));
    }
  } else {
    for (int64_t k = threadIdx.x; k < inner; k += blockDim.x) acc.add(__ldg(x + k) * __ldg(y + k));
  }
  __shared__ float red[8];
  float v = warp_sum(acc.s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    d.out[j][i * d.so[j]] = t;
  }
}
}  // namespace pfb

extern "C" int pfb_row_dots(int32_t n, const pfb_tensor* xs, const pfb_tensor* ys,
                            pfb_tensor* outs, void* stream) {
  using namespace pfb;
  if (n < 1 || n > kMaxDots) return PFB_E_ARG;
  RowDots d;
  d.n = n;
  d.rows = xs[0].shape[0];
  for (int j = 0; j < n; ++j) {
    const pfb_tensor *x = &xs[j], *y = &ys[j], *o = &outs[j];
    if (x->dtype != PFB_F32 || y->dtype != PFB_F32 || o->dtype != PFB_F32) return PFB_E_DTYPE;
    if (x->rank != 2 || y->rank != 2 || o->rank != 1) return PFB_E_RANK;
    if (x->shape[0] != d.rows || y->shape[0] != d.rows || o->shape[0] != d.rows ||
        x->shape[1] != y->shape[1])
      return PFB_E_SHAPE;
    if ((x->shape[1] > 1 && x->stride[1] != 1) || (y->shape[1] > 1 && y->stride[1] != 1))
      return PFB_E_UNSUPPORTED;
    d.x[j] = (const float*)x->data;
    d.y[j] = (const float*)y->data;
    d.inner[j] = x->shape[1];
    d.sx[j] = x->stride[0];
    d.sy[j] = y->stride[0];
    d.out[j] = (float*)o->data;
    d.so[j] = o->stride[0];
    d.vec[j] = (x->shape[1] % 4 == 0) && (d.sx[j] % 4 == 0) && (d.sy[j] % 4 == 0) &&
               (reinterpret_cast<uintptr_t>(x->data) % 16 == 0) &&
               (reinterpret_cast<uintptr_t>(y->data) % 16 == 0);
  }
  if (d.rows == 0) return 0;
  if (d.rows > 0x7fffffff) return PFB_E_UNSUPPORTED;
  launch(row_dots_kernel, dim3((unsigned)d.rows, (unsigned)n), 256, 0, as_stream(stream), d);
  return launch_status();
}

// ---------------------------------------------------------------------------
// Row sums of split-K partials (pass F15): out[i] = sum_s sum_k P_s[i, k] with
// P_s = x + s * part_stride ([rows, W], unit inner stride) -- the row
// reduction of a GEMM result that is still held as partials (cfg5's
// `reduce_sum(z) < 0` mask), so the partials need not be reduced into a
// tensor first.  One CTA per row; fixed per-thread order + tree: deterministic.

namespace pfb {
__global__ void __launch_bounds__(128) row_sum_parts_kernel(const float* __restrict__ x,
                                                            int64_t rs, int64_t W, int S,
                                                            int64_t ps, float* out, int64_t so) {
  pdl_enter();
  // one 128-thread CTA per row; its (partial, column) items spread over the
  // CTA in batches of 4 loads issued before they are added (cfg5: 8 partials
  // x 64 float4 = one batch per thread); fixed order, shuffle + smem tree
  const int64_t i = blockIdx.x;
  Acc<float> acc;
  const bool vec = (W % 4 == 0) && (rs % 4 == 0) && (ps % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const int64_t wv = vec ? W / 4 : W, items = (int64_t)S * wv;
  for (int64_t it0 = threadIdx.x; it0 < items; it0 += 4 * (int64_t)blockDim.x) {
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t it = it0 + u * (int64_t)blockDim.x;
      v[u] = 0.f;
      if (it < items) {
        const int64_t s = it / wv, k = it - s * wv;
        const float* r = x + s * ps + i * rs;
        if (vec) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(r) + k);
          v[u] = (a.x + a.y) + (a.z + a.w);
        } else {
          v[u] = __ldg(r + k);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc.add(v[u]);
  }
  __shared__ float red[4];
  const float v = warp_sum(acc.s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) out[i * so] = (red[0] + red[1]) + (red[2] + red[3]);
}
}  // namespace pfb

// ---------------------------------------------------------------------------
// Several weighted column sums in one launch (pass F19): out_q[c] =
// sum_r x_q[r, c] * y[r] for x_q [R, C_q] (any strides), y [R] -- the
// per-parameter-block bias-gradient sums of a clipped per-example gradient
// (sum_i s_i g_i, reference tensor.reduce_sum of a product, tensor.py:279-283)
// that share the clip scales.  A block = 32 columns x 8 row slices of one
// operand; the 8 slice sums are combined in slice order (deterministic).
namespace pfb {
constexpr int kMaxColDots = 8;
struct ColDots {
  const float* x[kMaxColDots];
  int64_t srow[kMaxColDots], scol[kMaxColDots];
  float* out[kMaxColDots];
  int64_t ncol[kMaxColDots];
  int64_t tile0[kMaxColDots + 1];  // first 32-column tile of operand q
};

__global__ void __launch_bounds__(256) col_dots_kernel(ColDots D, int q, int64_t R,
                                                       const float* y, int64_t sy) {
  pdl_enter();
  __shared__ float red[8][33];
  const int64_t tile = blockIdx.x;
  int o = 0;
  while (o + 1 < q && tile >= D.tile0[o + 1]) ++o;
  const int64_t c = (tile - D.tile0[o]) * 32 + (threadIdx.x & 31);
  const int slice = threadIdx.x >> 5;
  float acc = 0.f;
  if (c < D.ncol[o]) {
    const float* xp = D.x[o] + c * D.scol[o];
    for (int64_t r = slice; r < R; r += 8) acc = fmaf(__ldg(xp + r * D.srow[o]), __ldg(y + r * sy), acc);
  }
  red[slice][threadIdx.x & 31] = acc;
  __syncthreads();
  if (threadIdx.x < 32 && c < D.ncol[o]) {
    float t = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += red[k][threadIdx.x];
    D.out[o][c] = t;
  }
}
}  // namespace pfb

extern "C" int pfb_col_dots(int32_t q, const pfb_tensor* xs, const pfb_tensor* y, pfb_tensor* outs,
                            void* stream) {
  using namespace pfb;
  if (q < 1 || q > kMaxColDots) return PFB_E_ARG;
  if (y->dtype != PFB_F32) return PFB_E_DTYPE;
  // y: [R] or [R, 1] (any row stride)
  if (y->rank < 1 || y->rank > 2 || (y->rank == 2 && y->shape[1] != 1)) return PFB_E_SHAPE;
  const int64_t R = y->shape[0], sy = y->stride[0];
  ColDots D = {};
  int64_t tiles = 0;
  for (int k = 0; k < q; ++k) {
    const pfb_tensor& x = xs[k];
    const pfb_tensor& o = outs[k];
    if (x.dtype != PFB_F32 || o.dtype != PFB_F32) return PFB_E_DTYPE;
    if (x.rank != 2 || x.shape[0] != R || o.rank != 1 || o.shape[0] != x.shape[1] ||
        (o.shape[0] > 1 && o.stride[0] != 1))
      return PFB_E_SHAPE;
    D.x[k] = (const float*)x.data;
    D.srow[k] = x.stride[0];
    D.scol[k] = x.stride[1];
    D.out[k] = (float*)o.data;
    D.ncol[k] = x.shape[1];
    D.tile0[k] = tiles;
    tiles += (x.shape[1] + 31) / 32;
  }
  D.tile0[q] = tiles;
  if (tiles == 0) return 0;
  launch(col_dots_kernel, (unsigned)tiles, 256, 0, as_stream(stream), D, (int)q, R,
         (const float*)y->data, sy);
  return launch_status();
}

extern "C" int pfb_row_sum_parts(const pfb_tensor* x, int32_t parts, int64_t part_stride,
                                 pfb_tensor* out, void* stream) {
  using namespace pfb;
  if (x->dtype != PFB_F32 || out->dtype != PFB_F32) return PFB_E_DTYPE;
  if (x->rank != 2 || out->rank != 1 || out->shape[0] != x->shape[0] || parts < 1)
    return PFB_E_SHAPE;
  if (x->shape[1] > 1 && x->stride[1] != 1) return PFB_E_UNSUPPORTED;
  if (x->shape[0] == 0) return 0;
  launch(row_sum_parts_kernel, dim3((unsigned)x->shape[0]), dim3(128), 0, as_stream(stream),
         (const float*)x->data, x->stride[0], x->shape[1], (int)parts, part_stride,
         (float*)out->data, out->stride[0]);
  return launch_status();
}
