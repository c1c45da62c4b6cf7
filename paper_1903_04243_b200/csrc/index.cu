// Index kernels: gather / scatter / scatter-add / where_true / complement /
// iota / counter RNG.  Integer and index results are bit-exact with the
// reference (tensor.py:306-360, interp.py:52-82, 210-221); bounds, collision
// and cover violations set bits in a device error word instead of aborting.
#include "common.cuh"

namespace pfb {

// ---------------------------------------------------------------------------
// gather_rows: out[i, ...] = x[idx[i], ...]

// SEG (gather_stacked): index i belongs to segment i / seg, whose rows start
// at x + (i / seg) * seg_st -- out[j, q] = x[j, idx[j, q]], bounds [0, nrows)
template <typename T, bool VEC, bool SEG = false>
__global__ void __launch_bounds__(256) gather_kernel(Layout Lt, int64_t k, int64_t D,
                                                     const T* x, int64_t xrow, int64_t nrows,
                                                     const int64_t* idx, int64_t idx_st, T* out,
                                                     int64_t orow, int32_t* err, int64_t seg = 1,
                                                     int64_t seg_st = 0) {
  pdl_enter();
  const int64_t per = VEC ? D / 4 : D;
  const int64_t total = k * per;
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < total;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = lin / per, t = (lin - i * per) * (VEC ? 4 : 1);
    int64_t r = __ldg(idx + i * idx_st);
    bool ok = r >= 0 && r < nrows;
    if (!ok) set_err(err, PFB_DEV_OOB);
    if constexpr (SEG) r += (i / seg) * (seg_st / xrow);  // seg_st % xrow == 0 (checked)
    if (VEC) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (sizeof(T) == 4) {
        if (ok) v = __ldg(reinterpret_cast<const float4*>(x + r * xrow + t));
        *reinterpret_cast<float4*>(out + i * orow + t) = v;
      }
    } else {
      int64_t off[2];
      offsets<int64_t, 2>(Lt, t, off);
      out[i * orow + off[0]] = ok ? x[r * xrow + off[1]] : (T)0;
    }
  }
}

template <typename T>
int gather_run(const pfb_tensor* x, const pfb_tensor* idx, pfb_tensor* out, int32_t* err,
               cudaStream_t s) {
  int64_t k = idx->rank == 0 ? 1 : idx->shape[0];
  int64_t idx_st = idx->rank == 0 ? 0 : idx->stride[0];
  int tail_rank = x->rank - 1;
  int o0 = idx->rank == 0 ? 0 : 1;  // first tail dim of out
  if (out->rank != tail_rank + o0) return PFB_E_SHAPE;
  int64_t D = 1;
  for (int d = 0; d < tail_rank; ++d) {
    if (out->shape[o0 + d] != x->shape[1 + d]) return PFB_E_SHAPE;
    D *= x->shape[1 + d];
  }
  if (k == 0 || D == 0) return 0;
  const int64_t* st[2] = {out->stride + o0, x->stride + 1};
  Layout Lt = make_layout(tail_rank, x->shape + 1, 2, st);
  int64_t orow = idx->rank == 0 ? 0 : out->stride[0];
  bool vec = sizeof(T) == 4 && Lt.rank == 1 && Lt.st[0][0] == 1 && Lt.st[1][0] == 1 &&
             D % 4 == 0 && x->stride[0] % 4 == 0 && orow % 4 == 0 &&
             (uintptr_t)x->data % 16 == 0 && (uintptr_t)out->data % 16 == 0;
  int64_t work = k * (vec ? D / 4 : D);
  int grid = grid_for(work, 256);
  if (vec)
    launch(gather_kernel<T, true>, grid, 256, 0, s, Lt, k, D, (const T*)x->data, x->stride[0],
                                                 x->shape[0], (const int64_t*)idx->data, idx_st,
                                                 (T*)out->data, orow, err, (int64_t)1, (int64_t)0);
  else
    launch(gather_kernel<T, false>, grid, 256, 0, s, Lt, k, D, (const T*)x->data, x->stride[0],
                                                  x->shape[0], (const int64_t*)idx->data, idx_st,
                                                  (T*)out->data, orow, err, (int64_t)1, (int64_t)0);
  return launch_status();
}

// ---------------------------------------------------------------------------
// scatter_rows (disjoint cover) and scatter_add_rows (accumulating)

__global__ void count_rows(const int64_t* idx, int64_t st, int64_t k, int64_t total,
                           int32_t* cnt, int32_t* err) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx[i * st];
    if (r < 0 || r >= total) set_err(err, PFB_DEV_OOB);
    else atomicAdd(cnt + r, 1);
  }
}

__global__ void check_cover(const int32_t* cnt, int64_t total, int32_t* err) {
  pdl_enter();
  int32_t bits = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = cnt[i];
    if (c > 1) bits |= PFB_DEV_COLLISION;
    if (c == 0) bits |= PFB_DEV_COVER;
  }
  bits = __reduce_or_sync(0xffffffffu, bits);
  if (bits && (threadIdx.x & 31) == 0) set_err(err, bits);
}

// err != nullptr: an out-of-range row index is reported here (by the row's
// first element) instead of by a separate bounds-check launch
template <typename T, bool ADD>
__global__ void __launch_bounds__(256) scatter_kernel(Layout Lt, int64_t k, int64_t D,
                                                      const int64_t* idx, int64_t idx_st,
                                                      int64_t total, const T* src, int64_t srow,
                                                      T* out, int64_t orow, int32_t* err) {
  pdl_enter();
  const int64_t n = k * D;
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < n;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = lin / D, t = lin - i * D;
    int64_t r = idx[i * idx_st];
    if (r < 0 || r >= total) {
      if (t == 0) set_err(err, PFB_DEV_OOB);
      continue;
    }
    int64_t off[2];
    offsets<int64_t, 2>(Lt, t, off);
    T v = src[i * srow + off[1]];
    T* dst = out + r * orow + off[0];
    if constexpr (ADD) {
      if constexpr (std::is_same<T, int64_t>::value)
        atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)v);
      else
        atomicAdd(dst, v);
    } else {
      *dst = v;
    }
  }
}

__global__ void check_bounds(const int64_t* idx, int64_t st, int64_t k, int64_t total, int32_t* err) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx[i * st];
    if (r < 0 || r >= total) set_err(err, PFB_DEV_OOB);
  }
}

template <typename T, bool ADD>
int scatter_part(const pfb_tensor* idx, const pfb_tensor* src, int64_t total, pfb_tensor* out,
                 int32_t* err, cudaStream_t s) {
  int64_t k = idx->rank == 0 ? 1 : idx->shape[0];
  int64_t idx_st = idx->rank == 0 ? 0 : idx->stride[0];
  int s0 = idx->rank == 0 ? 0 : 1;  // first tail dim of src
  int tail_rank = out->rank - 1;
  if (src->rank != tail_rank + s0) return PFB_E_SHAPE;
  if (s0 && src->shape[0] != k) return PFB_E_SHAPE;
  int64_t D = 1;
  for (int d = 0; d < tail_rank; ++d) {
    if (src->shape[s0 + d] != out->shape[1 + d]) return PFB_E_SHAPE;
    D *= out->shape[1 + d];
  }
  if (k == 0) return 0;
  if (D == 0) {  // empty rows: nothing moves, the indices are still checked
    if (err) launch(check_bounds, grid_for(k, 256), 256, 0, s, (const int64_t*)idx->data, idx_st, k,
                    total, err);
    return launch_status();
  }
  const int64_t* st[2] = {out->stride + 1, src->stride + s0};
  Layout Lt = make_layout(tail_rank, out->shape + 1, 2, st);
  int64_t srow = s0 ? src->stride[0] : 0;
  launch(scatter_kernel<T, ADD>, grid_for(k * D, 256), 256, 0, s, 
      Lt, k, D, (const int64_t*)idx->data, idx_st, total, (const T*)src->data, srow,
      (T*)out->data, out->stride[0], err);
  return launch_status();
}

template <bool ADD>
int scatter_dispatch(const pfb_tensor* idx, const pfb_tensor* src, int64_t total, pfb_tensor* out,
                     int32_t* err, cudaStream_t s) {
  switch (out->dtype) {
    case PFB_F32: return scatter_part<float, ADD>(idx, src, total, out, err, s);
    case PFB_I64: return scatter_part<int64_t, ADD>(idx, src, total, out, err, s);
    default:
      if (ADD) return PFB_E_DTYPE;
      return scatter_part<uint8_t, false>(idx, src, total, out, err, s);
  }
}

// ---------------------------------------------------------------------------
// where_true: block-tiled stream compaction, ascending order

constexpr int kScanThreads = 1024;
constexpr int kScanPer = 4;
constexpr int kTile = kScanThreads * kScanPer;

__device__ __forceinline__ int block_exclusive_scan(int v, int* smem, int* total) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (blockDim.x >> 5) ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem[lane] = w;
  }
  __syncthreads();
  int base = warp ? smem[warp - 1] : 0;
  *total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return base + x - v;
}

// phase 1: per-tile counts
__global__ void __launch_bounds__(kScanThreads) tile_counts(const uint8_t* m, int64_t st, int64_t n,
                                                            int64_t* counts) {
  pdl_enter();
  __shared__ int smem[32];
  int64_t t0 = blockIdx.x * (int64_t)kTile + threadIdx.x * kScanPer;
  int c = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) c += (t0 + j < n) && m[(t0 + j) * st];
  int tot;
  block_exclusive_scan(c, smem, &tot);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

// phase 2: exclusive scan of tile counts (single block, loops)
__global__ void __launch_bounds__(kScanThreads) scan_counts(int64_t* counts, int64_t nt,
                                                            int64_t* dev_count) {
  pdl_enter();
  __shared__ int smem[32];
  int64_t carry = 0;
  for (int64_t b = 0; b < nt; b += kScanThreads) {
    int64_t i = b + threadIdx.x;
    int v = i < nt ? (int)counts[i] : 0;
    int tot;
    int ex = block_exclusive_scan(v, smem, &tot);
    if (i < nt) counts[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *dev_count = carry;
}

// phase 3: write indices
__global__ void __launch_bounds__(kScanThreads) tile_write(const uint8_t* m, int64_t st, int64_t n,
                                                           const int64_t* offs, int64_t* out,
                                                           int64_t* dev_count, int single) {
  pdl_enter();
  __shared__ int smem[32];
  int64_t t0 = blockIdx.x * (int64_t)kTile + threadIdx.x * kScanPer;
  uint8_t f[kScanPer];
  int c = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    f[j] = (t0 + j < n) && m[(t0 + j) * st];
    c += f[j];
  }
  int tot;
  int64_t pos = block_exclusive_scan(c, smem, &tot) + (single ? 0 : offs[blockIdx.x]);
#pragma unroll
  for (int j = 0; j < kScanPer; ++j)
    if (f[j]) out[pos++] = t0 + j;
  if (single && threadIdx.x == 0) *dev_count = tot;
}

int where_true_u8(const uint8_t* m, int64_t st, int64_t n, int64_t* out, int64_t* dev_count,
                  void* ws, int64_t ws_bytes, cudaStream_t s) {
  if (n == 0) {
    cudaMemsetAsync(dev_count, 0, sizeof(int64_t), s);
    return launch_status();
  }
  int64_t nt = (n + kTile - 1) / kTile;
  if (nt == 1) {
    launch(tile_write, 1, kScanThreads, 0, s, m, st, n, nullptr, out, dev_count, 1);
    return launch_status();
  }
  if (ws == nullptr || ws_bytes < nt * (int64_t)sizeof(int64_t)) return PFB_E_ARG;
  int64_t* counts = (int64_t*)ws;
  launch(tile_counts, (unsigned)nt, kScanThreads, 0, s, m, st, n, counts);
  launch(scan_counts, 1, kScanThreads, 0, s, counts, nt, dev_count);
  launch(tile_write, (unsigned)nt, kScanThreads, 0, s, m, st, n, counts, out, dev_count, 0);
  return launch_status();
}

__global__ void mark_kernel(uint8_t* mark, int64_t total, const int64_t* idx, int64_t st, int64_t k) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx[i * st];
    if (r >= 0 && r < total) mark[r] = 0;
  }
}

__global__ void iota_kernel(int64_t* out, int64_t n, int64_t start) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = start + i;
}

// ---------------------------------------------------------------------------
// splitmix64 counter stream (reference interp.py:52-82)

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

__global__ void rng_kernel(float* out, int64_t n, uint64_t dctr) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t bits = mix64(dctr ^ (uint64_t)i);
    out[i] = (float)((double)(bits >> 11) * 0x1.0p-53);
  }
}

}  // namespace pfb

using namespace pfb;

// gather_stacked (x [n, m, ...], idx [n] or [n, q]): out[j, (q,) ...] =
// x[j, idx[j, (q)], ...] -- pfor's gather with a stacked operand AND a stacked
// index in one launch (the reference falls back to a sequential loop,
// vectorize.py:271-273); an index outside [0, m) sets PFB_DEV_OOB.
template <typename T>
int gather_stacked_run(const pfb_tensor* x, const pfb_tensor* idx, pfb_tensor* out, int32_t* err,
                       cudaStream_t s) {
  const int64_t n = x->shape[0], m = x->shape[1];
  const int64_t q = idx->rank == 2 ? idx->shape[1] : 1;
  if (idx->shape[0] != n) return PFB_E_SHAPE;
  if (idx->rank == 2 && q > 1 && idx->stride[0] != q * idx->stride[1]) return PFB_E_UNSUPPORTED;
  const int64_t idx_st = idx->rank == 2 ? idx->stride[1] : idx->stride[0];
  const int tail_rank = x->rank - 2;
  const int o0 = idx->rank;  // first tail dim of out
  if (out->rank != tail_rank + o0 || out->shape[0] != n || (idx->rank == 2 && out->shape[1] != q))
    return PFB_E_SHAPE;
  int64_t D = 1;
  for (int d = 0; d < tail_rank; ++d) {
    if (out->shape[o0 + d] != x->shape[2 + d]) return PFB_E_SHAPE;
    D *= x->shape[2 + d];
  }
  // out rows [n * q] must be one stride apart; x's segment stride a multiple of its row stride
  const int64_t orow = out->stride[o0 - 1];
  if (idx->rank == 2 && q > 1 && out->stride[0] != q * orow) return PFB_E_UNSUPPORTED;
  const int64_t xrow = x->stride[1];
  if (n * q == 0 || D == 0) return 0;
  if (xrow == 0 || x->stride[0] % xrow != 0) return PFB_E_UNSUPPORTED;
  int64_t tail_shape[kMaxRank];
  for (int d = 0; d < tail_rank; ++d) tail_shape[d] = x->shape[2 + d];
  const int64_t* st[2] = {out->stride + o0, x->stride + 2};
  Layout Lt = make_layout(tail_rank, tail_shape, 2, st);
  const bool vec = sizeof(T) == 4 && Lt.rank == 1 && Lt.st[0][0] == 1 && Lt.st[1][0] == 1 &&
                   D % 4 == 0 && xrow % 4 == 0 && x->stride[0] % 4 == 0 && orow % 4 == 0 &&
                   (uintptr_t)x->data % 16 == 0 && (uintptr_t)out->data % 16 == 0;
  const int64_t k = n * q;
  const int grid = grid_for(k * (vec ? D / 4 : D), 256);
  if (vec)
    launch(gather_kernel<T, true, true>, grid, 256, 0, s, Lt, k, D, (const T*)x->data, xrow, m,
           (const int64_t*)idx->data, idx_st, (T*)out->data, orow, err, (int64_t)q, (int64_t)x->stride[0]);
  else
    launch(gather_kernel<T, false, true>, grid, 256, 0, s, Lt, k, D, (const T*)x->data, xrow, m,
           (const int64_t*)idx->data, idx_st, (T*)out->data, orow, err, (int64_t)q, (int64_t)x->stride[0]);
  return launch_status();
}

extern "C" int pfb_gather_stacked(const pfb_tensor* x, const pfb_tensor* idx, pfb_tensor* out,
                                  int32_t* dev_err, void* stream) {
  if (idx->dtype != PFB_I64) return PFB_E_DTYPE;
  if (idx->rank < 1 || idx->rank > 2 || x->rank < 2) return PFB_E_RANK;
  if (x->dtype != out->dtype) return PFB_E_DTYPE;
  cudaStream_t s = as_stream(stream);
  switch (x->dtype) {
    case PFB_F32: return gather_stacked_run<float>(x, idx, out, dev_err, s);
    case PFB_I64: return gather_stacked_run<int64_t>(x, idx, out, dev_err, s);
    default: return gather_stacked_run<uint8_t>(x, idx, out, dev_err, s);
  }
}

// several gather_stacked of one operand (pass F17: the per-step x_t gathers
// of an unrolled loop body) in one launch: out_g[j, :] = x[j, idx_g[j], :],
// g = 0..q-1, each index vector with its own error word.  fp32 rows with a
// contiguous 16-byte-aligned tail only (128-bit accesses); anything else is
// PFB_E_UNSUPPORTED (the caller then gathers one index vector at a time).
namespace pfb {
constexpr int kMaxGathers = 8;
struct GatherMany {
  const int64_t* idx[kMaxGathers];
  int64_t idx_st[kMaxGathers];
  float* out[kMaxGathers];
  int64_t orow[kMaxGathers];
  int32_t* err[kMaxGathers];
};

__global__ void __launch_bounds__(256) gather_many_kernel(int q, int64_t n, int64_t per,
                                                          const float* x, int64_t xrow,
                                                          int64_t xseg, int64_t m, GatherMany G) {
  pdl_enter();
  const int64_t rows = (int64_t)q * n, total = rows * per;
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < total;
       lin += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = lin / per, t = (lin - rr * per) * 4;
    const int g = (int)(rr / n);
    const int64_t j = rr - (int64_t)g * n;
    const int64_t r = __ldg(G.idx[g] + j * G.idx_st[g]);
    const bool ok = r >= 0 && r < m;
    if (!ok) set_err(G.err[g], PFB_DEV_OOB);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok) v = __ldg(reinterpret_cast<const float4*>(x + j * xseg + r * xrow + t));
    *reinterpret_cast<float4*>(G.out[g] + j * G.orow[g] + t) = v;
  }
}
}  // namespace pfb

extern "C" int pfb_gather_stacked_many(const pfb_tensor* x, int32_t q, const pfb_tensor* idx,
                                       pfb_tensor* out, int32_t* const* dev_err, void* stream) {
  if (q < 1 || q > kMaxGathers) return PFB_E_ARG;
  if (x->rank < 2) return PFB_E_RANK;
  if (x->dtype != PFB_F32) return PFB_E_UNSUPPORTED;
  const int64_t n = x->shape[0], m = x->shape[1];
  int64_t D = 1;
  for (int d = 2; d < x->rank; ++d) D *= x->shape[d];
  // x's tail contiguous (one row of D elements per (j, r))
  int64_t e = 1;
  for (int d = x->rank - 1; d >= 2; --d) {
    if (x->shape[d] != 1 && x->stride[d] != e) return PFB_E_UNSUPPORTED;
    e *= x->shape[d];
  }
  const int64_t xrow = x->stride[1], xseg = x->stride[0];
  if (D % 4 || xrow % 4 || xseg % 4 || (uintptr_t)x->data % 16) return PFB_E_UNSUPPORTED;
  GatherMany G;
  for (int g = 0; g < q; ++g) {
    const pfb_tensor& I = idx[g];
    const pfb_tensor& O = out[g];
    if (I.dtype != PFB_I64) return PFB_E_DTYPE;
    if (I.rank != 1 || I.shape[0] != n) return PFB_E_SHAPE;
    if (O.dtype != PFB_F32 || O.rank != x->rank - 1 || O.shape[0] != n) return PFB_E_SHAPE;
    int64_t eo = 1;
    for (int d = O.rank - 1; d >= 1; --d) {
      if (O.shape[d] != x->shape[d + 1]) return PFB_E_SHAPE;
      if (O.shape[d] != 1 && O.stride[d] != eo) return PFB_E_UNSUPPORTED;
      eo *= O.shape[d];
    }
    const int64_t orow = O.rank == 1 ? 0 : O.stride[0];
    if ((O.rank > 1 && orow % 4) || (uintptr_t)O.data % 16) return PFB_E_UNSUPPORTED;
    G.idx[g] = (const int64_t*)I.data;
    G.idx_st[g] = I.stride[0];
    G.out[g] = (float*)O.data;
    G.orow[g] = orow;
    G.err[g] = dev_err ? dev_err[g] : nullptr;
  }
  if (n == 0 || D == 0) return 0;
  const int64_t per = D / 4;
  cudaStream_t s = as_stream(stream);
  launch(gather_many_kernel, grid_for((int64_t)q * n * per, 256), 256, 0, s, (int)q, n, per,
         (const float*)x->data, xrow, xseg, m, G);
  return launch_status();
}

extern "C" int pfb_gather_rows(const pfb_tensor* x, const pfb_tensor* idx, pfb_tensor* out,
                               int32_t* dev_err, void* stream) {
  if (idx->dtype != PFB_I64) return PFB_E_DTYPE;
  if (idx->rank > 1) return PFB_E_RANK;
  if (x->rank == 0) return PFB_E_RANK;
  if (x->dtype != out->dtype) return PFB_E_DTYPE;
  cudaStream_t s = as_stream(stream);
  switch (x->dtype) {
    case PFB_F32: return gather_run<float>(x, idx, out, dev_err, s);
    case PFB_I64: return gather_run<int64_t>(x, idx, out, dev_err, s);
    default: return gather_run<uint8_t>(x, idx, out, dev_err, s);
  }
}

extern "C" int pfb_scatter_rows(int32_t n_parts, const pfb_tensor* index_sets,
                                const pfb_tensor* parts, int64_t total, pfb_tensor* out,
                                int32_t* ws_count, int32_t* dev_err, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (total > 0) {
    cudaMemsetAsync(ws_count, 0, total * sizeof(int32_t), s);
    for (int p = 0; p < n_parts; ++p) {
      const pfb_tensor* ix = &index_sets[p];
      int64_t k = ix->rank == 0 ? 1 : ix->shape[0];
      if (k == 0) continue;
      launch(count_rows, grid_for(k, 256), 256, 0, s, (const int64_t*)ix->data,
                                                 ix->rank ? ix->stride[0] : 0, k, total,
                                                 ws_count, dev_err);
    }
    launch(check_cover, grid_for(total, 256), 256, 0, s, ws_count, total, dev_err);
  }
  // (total == 0: every index is out of range; the scatter kernels report it)
  for (int p = 0; p < n_parts; ++p) {
    if (int e = scatter_dispatch<false>(&index_sets[p], &parts[p], total, out,
                                        total > 0 ? nullptr : dev_err, s))
      return e;
  }
  return launch_status();
}

extern "C" int pfb_scatter_add_rows(const pfb_tensor* idx, const pfb_tensor* updates, int64_t total,
                                    pfb_tensor* out, int32_t* dev_err, void* stream) {
  if (idx->dtype != PFB_I64) return PFB_E_DTYPE;
  if (!is_dense(out)) return PFB_E_UNSUPPORTED;
  cudaStream_t s = as_stream(stream);
  int64_t n = numel(out);
  if (n) cudaMemsetAsync(out->data, 0, n * dtype_size(out->dtype), s);
  // index bounds are checked inside the scatter kernel (one launch)
  if (int e = scatter_dispatch<true>(idx, updates, total, out, dev_err, s)) return e;
  return launch_status();
}

extern "C" int pfb_where_true(const pfb_tensor* mask, pfb_tensor* out, int64_t* dev_count, void* ws,
                              int64_t ws_bytes, void* stream) {
  if (mask->dtype != PFB_BOOL || mask->rank != 1) return PFB_E_DTYPE;
  if (out->dtype != PFB_I64) return PFB_E_DTYPE;
  return where_true_u8((const uint8_t*)mask->data, mask->stride[0], mask->shape[0],
                       (int64_t*)out->data, dev_count, ws, ws_bytes, as_stream(stream));
}

extern "C" int pfb_complement(const pfb_tensor* idx, int64_t total, pfb_tensor* out,
                              int64_t* dev_count, void* ws, int64_t ws_bytes, void* stream) {
  if (idx->dtype != PFB_I64 || idx->rank > 1) return PFB_E_DTYPE;
  cudaStream_t s = as_stream(stream);
  if (total <= 0) {
    cudaMemsetAsync(dev_count, 0, sizeof(int64_t), s);
    return launch_status();
  }
  int64_t mark_bytes = (total + 255) / 256 * 256;
  if (ws == nullptr || ws_bytes < mark_bytes) return PFB_E_ARG;
  uint8_t* mark = (uint8_t*)ws;
  cudaMemsetAsync(mark, 1, total, s);
  int64_t k = idx->rank == 0 ? 1 : idx->shape[0];
  if (k) launch(mark_kernel, grid_for(k, 256), 256, 0, s, mark, total, (const int64_t*)idx->data,
                                                      idx->rank ? idx->stride[0] : 0, k);
  return where_true_u8(mark, 1, total, (int64_t*)out->data, dev_count, (char*)ws + mark_bytes,
                       ws_bytes - mark_bytes, s);
}

extern "C" int pfb_iota(pfb_tensor* out, int64_t start, void* stream) {
  if (out->dtype != PFB_I64 || !is_dense(out)) return PFB_E_DTYPE;
  int64_t n = numel(out);
  if (n == 0) return 0;
  launch(iota_kernel, grid_for(n, 256), 256, 0, as_stream(stream), (int64_t*)out->data, n, start);
  return launch_status();
}

extern "C" int pfb_rng_uniform(uint64_t seed, uint64_t counter, pfb_tensor* out, void* stream) {
  if (out->dtype != PFB_F32 || !is_dense(out)) return PFB_E_DTYPE;
  int64_t n = numel(out);
  if (n == 0) return 0;
  uint64_t dctr = mix64(mix64(seed) ^ counter);
  launch(rng_kernel, grid_for(n, 256), 256, 0, as_stream(stream), (float*)out->data, n, dctr);
  return launch_status();
}
