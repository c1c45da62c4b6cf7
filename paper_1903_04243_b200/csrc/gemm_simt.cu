// SIMT fp32 GEMM for shapes the tensor-core path does not take: tiny K
// (K=1 outer products, K=10 cotangents), skinny M (batch-32 forward passes),
// tiny per-example conv filter grads (9x8) and odd strides.
//
//  * tile kernel: 64x64x16 tiles, 256 threads, 4x4 register micro-tile;
//    operands staged through shared memory with the global read mapped onto
//    whichever of their two strides is unit (coalesced for normal and
//    transposed views); 128-bit stores of 4 consecutive output columns.
//    Split-K (grid.z = batch x splits) when there are too few tiles to fill
//    148 SMs: the splits of a tile form one thread-block cluster; each CTA
//    leaves its partial tile in shared memory and, after a cluster barrier,
//    CTA r sums rows [r*64/S, (r+1)*64/S) of all S partials over DSMEM in
//    split order (deterministic) and applies the epilogue -- one launch, no
//    workspace.  (Splits beyond the cluster limit: partials to the workspace
//    and a second pass.)
//  * small-K kernel (K <= 16): store-bound; a CTA per output row, each thread
//    4 consecutive columns per 128-bit store, the row's lhs in registers.
// Exact fp32 FMA accumulation in both.
#include <algorithm>

#include "gemm.cuh"

namespace pfb {

constexpr int BM = 64, BN = 64, BK = 16;

__device__ __forceinline__ void store_row4(const GemmArgs& g, int64_t b, int64_t m, int64_t n,
                                           const float* v, float alpha) {
  if (m >= g.M) return;
  float* p = g.C + b * g.scb + m * g.scm + n * g.scn;
  if (g.scn == 1 && n + 3 < g.N && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    float4 o = make_float4(v[0] * alpha, v[1] * alpha, v[2] * alpha, v[3] * alpha);
    if (g.accumulate) {
      float4 c = *reinterpret_cast<float4*>(p);
      o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
    }
    if (g.has_epi()) {
      o.x = epi_value(g, b, m, n, o.x); o.y = epi_value(g, b, m, n + 1, o.y);
      o.z = epi_value(g, b, m, n + 2, o.z); o.w = epi_value(g, b, m, n + 3, o.w);
    }
    *reinterpret_cast<float4*>(p) = o;
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (n + j >= g.N) break;
    float* q = p + j * g.scn;
    float x = v[j] * alpha;
    if (g.accumulate) x += *q;
    *q = epi_value(g, b, m, n + j, x);
  }
}

// partials: nullptr -> epilogue straight to C; else ws[split][b][M][N].
// Register-staged double buffering: the next k-tile's global loads are issued
// before the current tile's FMAs, so the loop is not load-latency bound.
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool pred) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gmem),
               "r"(pred ? 4 : 0)
               : "memory");
}

constexpr int NST = 4;  // k-tiles in flight (cp.async ring)

// split-K tile tickets of the workspace path (last split reduces); every
// launch leaves them zero.  One stream at a time per process uses them (the
// executor's), so a launch never shares a ticket with a concurrent one.
constexpr unsigned kSimtTiles = 1u << 16;
__device__ unsigned g_simt_tiles[kSimtTiles];

template <bool KS, bool CL>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g, int splits, int64_t kchunk,
                                                        float* partials, bool tile_reduce) {
  pdl_enter();
  // NST-deep cp.async ring of A/B k-tiles: a CTA's whole K range (<= 4
  // k-tiles for split-K shapes) is requested at once, so a small GEMM pays
  // one memory latency instead of one per k-tile.  (The cluster reduction
  // buffer aliases the ring after the main loop.)
  __shared__ __align__(16) float ring[NST * 2 * BK * (BM + 4)];
  __shared__ float ks_s[NST][BK];
  auto As = [&](int st) { return ring + st * 2 * BK * (BM + 4); };
  auto Bs = [&](int st) { return ring + st * 2 * BK * (BM + 4) + BK * (BM + 4); };
  const int64_t bz = blockIdx.z / splits;
  const int split = blockIdx.z % splits;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = split * kchunk, kend = std::min<int64_t>(g.K, kbeg + kchunk);
  const float* A = g.A + bz * g.sab;
  const float* B = g.B + bz * g.sbb;
  const int tid = threadIdx.x;
  const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
  float acc[4][4] = {};
  const bool a_kfast = g.sak == 1 || g.sam != 1;
  const bool b_nfast = g.sbn == 1 || g.sbk != 1;
  int am[4], ak[4], bk[4], bn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e = tid + j * 256;
    if (a_kfast) { am[j] = e / BK; ak[j] = e % BK; } else { ak[j] = e / BM; am[j] = e % BM; }
    if (b_nfast) { bk[j] = e / BN; bn[j] = e % BN; } else { bn[j] = e / BK; bk[j] = e % BK; }
  }
  const int ntiles = kbeg < kend ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  auto issue = [&](int t) {  // k-tile t -> ring stage t % NST (one commit group)
    const int st = t % NST;
    const int64_t k0 = kbeg + (int64_t)t * BK;
    float* as = As(st);
    float* bs = Bs(st);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gm = m0 + am[j], gk = k0 + ak[j];
      const bool pa = gm < g.M && gk < kend;
      cp_async4(as + ak[j] * (BM + 4) + am[j], pa ? A + gm * g.sam + gk * g.sak : A, pa);
      const int64_t gk2 = k0 + bk[j], gn = n0 + bn[j];
      const bool pb = gk2 < kend && gn < g.N;
      cp_async4(bs + bk[j] * (BN + 4) + bn[j], pb ? B + gk2 * g.sbk + gn * g.sbn : B, pb);
    }
    if (KS && tid < BK) {
      const int64_t gk = k0 + tid;
      const bool pk = gk < kend;
      cp_async4(&ks_s[st][tid], pk ? g.kscale + bz * g.skb + gk * g.skk : g.kscale, pk);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int t = 0; t < NST - 1; ++t) {
    if (t < ntiles) issue(t);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int t = 0; t < ntiles; ++t) {
    if (t + NST - 1 < ntiles) issue(t + NST - 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
    __syncthreads();
    const float* as = As(t % NST);
    const float* bs = Bs(t % NST);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 a4 = *reinterpret_cast<const float4*>(as + kk * (BM + 4) + tm);
      const float4 b4 = *reinterpret_cast<const float4*>(bs + kk * (BN + 4) + tn);
      if (KS) {
        const float sc = ks_s[t % NST][kk];
        a4.x *= sc; a4.y *= sc; a4.z *= sc; a4.w *= sc;
      }
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if constexpr (CL) {
    // cluster split-K: partial tile -> own smem, DSMEM reduction in split order
    float* red = ring;  // BM*BN floats, the (drained) ring
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(&red[(tm + i) * BN + tn]) =
          make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                     "memory");
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int rows_per = (BM + splits - 1) / splits;
    const int rb = (int)rank * rows_per, re = min((int)BM, rb + rows_per);
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(red));
    for (int idx = tid; idx < (re - rb) * (BN / 4); idx += 256) {
      const int row = rb + idx / (BN / 4), c4 = idx % (BN / 4);
      const uint32_t off = base + (uint32_t)(row * BN + 4 * c4) * 4u;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      for (int q = 0; q < splits; ++q) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(off), "r"(q));
        float x0, x1, x2, x3;
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3)
                     : "r"(remote)
                     : "memory");
        v[0] += x0; v[1] += x1; v[2] += x2; v[3] += x3;
      }
      const int64_t gm = m0 + row;
      if (gm < g.M && n0 + 4 * c4 < g.N) {
        const float alpha = g.alpha_rows ? g.alpha_rows[bz * g.M + gm] : 1.f;
        store_row4(g, bz, gm, n0 + 4 * c4, v, alpha);
      }
    }
    // peers' shared memory stays live until every CTA has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                     "memory");
  } else if (partials == nullptr) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t gm = m0 + tm + i;
      const float alpha = (g.alpha_rows && gm < g.M) ? g.alpha_rows[bz * g.M + gm] : 1.f;
      store_row4(g, bz, gm, n0 + tn, acc[i], alpha);
    }
  } else {
    float* P = partials + ((int64_t)split * g.batch + bz) * g.M * g.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t gm = m0 + tm + i;
      if (gm >= g.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (n0 + tn + j < g.N) P[gm * g.N + n0 + tn + j] = acc[i][j];
    }
    // the last split of this tile to finish sums all partials of the tile in
    // split order (the reduce kernel's order: deterministic) and applies the
    // epilogue -- no second launch.  Tile tickets wrap to 0 (atomicInc), so
    // the counters are clean for the next launch.
    if (!tile_reduce) return;
    __shared__ unsigned last;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const unsigned tile = ((unsigned)bz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      last = atomicInc(&g_simt_tiles[tile], (unsigned)splits - 1) == (unsigned)splits - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      const int64_t per = g.M * g.N, total = g.batch * per;
      for (int e = tid; e < BM * BN; e += 256) {
        const int64_t gm = m0 + e / BN, gn = n0 + e % BN;
        if (gm >= g.M || gn >= g.N) continue;
        const int64_t off = bz * per + gm * g.N + gn;
        float v = 0.f;
        for (int q = 0; q < splits; ++q) v += __ldcg(partials + (int64_t)q * total + off);
        if (g.alpha_rows) v *= g.alpha_rows[bz * g.M + gm];
        float* c = g.C + bz * g.scb + gm * g.scm + gn * g.scn;
        if (g.accumulate) v += *c;
        *c = epi_value(g, bz, gm, gn, v);
      }
    }
  }
}

// sum split partials in split order (deterministic); 32-bit indexing, the
// split loop unrolled so its loads are in flight together
__global__ void __launch_bounds__(256) splitk_reduce(GemmArgs g, int splits, const float* partials) {
  pdl_enter();
  const uint32_t N = (uint32_t)g.N, per = (uint32_t)(g.M * g.N);
  const uint32_t total = (uint32_t)(g.batch * g.M * g.N);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    float s = 0.f;
#pragma unroll 8
    for (int k = 0; k < splits; ++k) s += __ldg(partials + (size_t)k * total + i);
    const uint32_t b = i / per, r = i - b * per;
    const uint32_t m = r / N, n = r - m * N;
    if (g.alpha_rows) s *= g.alpha_rows[(size_t)b * g.M + m];
    float* p = g.C + b * g.scb + m * g.scm + n * g.scn;
    if (g.accumulate) s += *p;
    *p = epi_value(g, b, m, n, s);
  }
}

// K <= 16 (outer products, K=1 weight jacobians): store-bound.  One CTA per
// output row at a time (grid-stride over rows); the row's K lhs values are
// read once into registers, every thread then produces 4 consecutive columns
// per iteration with one 128-bit store -- a warp writes 512 contiguous bytes.
template <bool VEC>
__global__ void __launch_bounds__(256) gemm_smallk_kernel(GemmArgs g) {
  pdl_enter();
  const int64_t rows = g.batch * g.M;
  const int64_t nq = (g.N + 3) / 4;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t b = row / g.M, m = row - b * g.M;
    float av[16];
    const float* a = g.A + b * g.sab + m * g.sam;
#pragma unroll
    for (int k = 0; k < 16; ++k) av[k] = k < g.K ? __ldg(a + k * g.sak) * kscale_at(g, b, k) : 0.f;
    const float alpha = g.alpha_rows ? g.alpha_rows[row] : 1.f;
    const float* bb = g.B + b * g.sbb;
    float* crow = g.C + b * g.scb + m * g.scm;
    for (int64_t q = threadIdx.x; q < nq; q += blockDim.x) {
      const int64_t n = q * 4;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (VEC) {
#pragma unroll 4
        for (int k = 0; k < g.K; ++k) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(bb + k * g.sbk + n));
          acc[0] = fmaf(av[k], v.x, acc[0]); acc[1] = fmaf(av[k], v.y, acc[1]);
          acc[2] = fmaf(av[k], v.z, acc[2]); acc[3] = fmaf(av[k], v.w, acc[3]);
        }
        float4 o = make_float4(acc[0] * alpha, acc[1] * alpha, acc[2] * alpha, acc[3] * alpha);
        float4* dst = reinterpret_cast<float4*>(crow + n);
        if (g.accumulate) {
          const float4 c = *dst;
          o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
        }
        if (g.has_epi()) {
          o.x = epi_value(g, b, m, n, o.x); o.y = epi_value(g, b, m, n + 1, o.y);
          o.z = epi_value(g, b, m, n + 2, o.z); o.w = epi_value(g, b, m, n + 3, o.w);
        }
        if (g.accumulate) *dst = o;
        else __stcs(dst, o);  // write-once output (jacobian rows): streaming store
      } else {
        for (int k = 0; k < g.K; ++k) {
          const float* bk = bb + k * g.sbk + n * g.sbn;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (n + j < g.N) acc[j] = fmaf(av[k], __ldg(bk + j * g.sbn), acc[j]);
        }
        store_row4(g, b, m, n, acc, alpha);
      }
    }
  }
}

// K = 1, rhs unit-stride: C[b, m, :] = a[b, m] * B[b, 0, :].  Each thread owns
// 4 consecutive columns (kept in registers) and streams a block of rows with
// 128-bit streaming stores -- the cfg3 weight-jacobian writer (store-bound).
__global__ void __launch_bounds__(256) outer1_kernel(GemmArgs g, int64_t rows_per_cta) {
  pdl_enter();
  const int64_t nq = g.N / 4;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int64_t rows = g.batch * g.M;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r1 = r0 + rows_per_cta < rows ? r0 + rows_per_cta : rows;
  int64_t b = r0 / g.M, m = r0 - b * g.M;
  float4 bv = __ldg(reinterpret_cast<const float4*>(g.B + b * g.sbb) + q);
  for (int64_t r = r0; r < r1; ++r) {
    const float av = __ldg(g.A + b * g.sab + m * g.sam) * kscale_at(g, b, 0);
    const float alpha = g.alpha_rows ? g.alpha_rows[r] : 1.f;
    float4* dst = reinterpret_cast<float4*>(g.C + b * g.scb + m * g.scm) + q;
    float4 o = make_float4(av * bv.x * alpha, av * bv.y * alpha, av * bv.z * alpha,
                           av * bv.w * alpha);
    if (g.accumulate) {
      const float4 c = *dst;
      o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
    }
    if (g.has_epi()) {
      const int64_t n = 4 * q;
      o.x = epi_value(g, b, m, n, o.x); o.y = epi_value(g, b, m, n + 1, o.y);
      o.z = epi_value(g, b, m, n + 2, o.z); o.w = epi_value(g, b, m, n + 3, o.w);
    }
    if (g.accumulate) *dst = o;
    else __stcs(dst, o);
    if (++m == g.M) {
      m = 0;
      ++b;
      if (r + 1 < r1) bv = __ldg(reinterpret_cast<const float4*>(g.B + b * g.sbb) + q);
    }
  }
}

// N <= 16 (logits layers, class-dimension cotangents: cfg2's h W2 and
// h^T diag(s) dlogits): one warp per output row, lanes stride over K with
// all N accumulators in registers, then a fixed-order shuffle reduction per
// column -- a 64x64 tile would leave 84% of its lanes idle and still need
// split-K for parallelism.
template <int NMAX, bool KS>
__global__ void __launch_bounds__(256) gemm_narrow_kernel(GemmArgs g, int wpr) {
  // wpr warps per output row split K (each a contiguous K range); their
  // partial sums meet in shared memory in warp order (deterministic)
  pdl_enter();
  __shared__ float part[8][NMAX];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rows_per_block = 8 / wpr;
  const int64_t rows = g.batch * g.M;
  const int64_t row = (int64_t)blockIdx.x * rows_per_block + w / wpr;
  const int sub = w % wpr;
  const bool live = row < rows;
  const int64_t b = live ? row / g.M : 0, m = live ? row - b * g.M : 0;
  const int64_t kchunk = (g.K + wpr - 1) / wpr;
  const int64_t k0 = sub * kchunk, k1 = live ? min(g.K, k0 + kchunk) : 0;
  const float* A = g.A + b * g.sab + m * g.sam;
  const float* B = g.B + b * g.sbb;
  float acc[NMAX];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) acc[j] = 0.f;
  // 4 k per lane per trip: all their loads are in flight together
  int64_t k = k0 + lane;
  for (; k + 96 < k1; k += 128) {
    float a[4];
    float bv[4][NMAX];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t ku = k + 32 * u;
      a[u] = __ldg(A + ku * g.sak);
      if (KS) a[u] *= __ldg(g.kscale + b * g.skb + ku * g.skk);
#pragma unroll
      for (int j = 0; j < NMAX; ++j) bv[u][j] = j < g.N ? __ldg(B + ku * g.sbk + j * g.sbn) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < NMAX; ++j) acc[j] = fmaf(a[u], bv[u][j], acc[j]);
  }
  for (; k < k1; k += 32) {
    float a = __ldg(A + k * g.sak);
    if (KS) a *= __ldg(g.kscale + b * g.skb + k * g.skk);
    const float* bk = B + k * g.sbk;
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
      if (j < g.N) acc[j] = fmaf(a, __ldg(bk + j * g.sbn), acc[j]);
  }
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  }
  float v = 0.f;
#pragma unroll
  for (int j = 0; j < NMAX; ++j)
    if (lane == j) v = acc[j];
  if (wpr > 1) {
    if (lane < NMAX) part[w][lane] = v;
    __syncthreads();
    if (sub != 0) return;
    for (int q = 1; q < wpr; ++q) v += lane < NMAX ? part[w + q][lane] : 0.f;
  }
  if (live && lane < g.N) {
    float* p = g.C + b * g.scb + m * g.scm + lane * g.scn;
    float x = v * (g.alpha_rows ? g.alpha_rows[row] : 1.f);
    if (g.accumulate) x += *p;
    *p = epi_value(g, b, m, lane, x);
  }
}

static int narrow_launch(const GemmArgs& g, cudaStream_t s) {
  const int64_t rows = g.batch * g.M;
  // warps per row: keep each warp's K range within ~128 (one unrolled trip)
  // while there are few rows to spread over the SMs
  int wpr = 1;
  while (wpr < 8 && g.K > 128 * wpr && rows * wpr < (int64_t)kNumSMs * 16) wpr *= 2;
  const int64_t blocks = (rows * wpr + 7) / 8;
  if (blocks > 0x7fffffff) return PFB_E_UNSUPPORTED;
  if (g.kscale) launch(gemm_narrow_kernel<16, true>, (unsigned)blocks, 256, 0, s, g, wpr);
  else launch(gemm_narrow_kernel<16, false>, (unsigned)blocks, 256, 0, s, g, wpr);
  return launch_status();
}

static int smallk_launch(const GemmArgs& g, cudaStream_t s) {
  const bool vec = g.K <= 16 && g.sbn == 1 && g.scn == 1 && g.N % 4 == 0 && g.sbk % 4 == 0 &&
                   g.sbb % 4 == 0 && g.scm % 4 == 0 && g.scb % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(g.B) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(g.C) & 15) == 0;
  const int64_t rows = g.batch * g.M;
  if (vec && g.K == 1 && g.N >= 512) {
    const int64_t nq = g.N / 4;
    const unsigned gx = (unsigned)((nq + 255) / 256);
    // enough CTAs for ~8 per SM, at least 16 rows each
    int64_t rpc = std::max<int64_t>(16, rows * gx / ((int64_t)kNumSMs * 8));
    const int64_t gy = (rows + rpc - 1) / rpc;
    if (gy <= 65535) {
      launch(outer1_kernel, dim3(gx, (unsigned)gy), 256, 0, s, g, rpc);
      return launch_status();
    }
  }
  const int grid = (int)std::min<int64_t>(rows, (int64_t)kNumSMs * 8);
  if (vec) launch(gemm_smallk_kernel<true>, grid, 256, 0, s, g);
  else launch(gemm_smallk_kernel<false>, grid, 256, 0, s, g);
  return launch_status();
}

static int simt_splits(const GemmArgs& g) {
  if ((int64_t)g.batch * g.M * g.N >= 0x7fffffff) return 1;  // 32-bit reduction indexing
  const int64_t tiles = ((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM) * g.batch;
  if (tiles >= kNumSMs || g.K < 64) return 1;
  // aim for >= 148 CTAs with >= 2 k-tiles (32) each; a split-K group is one
  // cluster (<= 16 CTAs), so the reduction stays on chip
  int64_t s = (kNumSMs + tiles - 1) / tiles;
  s = std::min<int64_t>(s, g.K / 32);
  s = std::min<int64_t>(s, 16);
  if (const char* e = getenv("PFB_SIMT_SPLITS")) s = atoi(e);  // experiments
  return (int)std::max<int64_t>(s, 1);
}

constexpr int kMaxSimtCluster = 16;  // non-portable cluster size (B200 supports 16)
constexpr int kSimtWsSplits = 16;    // autotuner candidate: k-splits reduced through the workspace

static bool cluster16_ok() {
  static int ok = -1;
  if (ok < 0) {
    ok = cudaFuncSetAttribute(gemm_simt_kernel<false, true>,
                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
         cudaFuncSetAttribute(gemm_simt_kernel<true, true>,
                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    cudaGetLastError();
  }
  return ok == 1;
}

static int cluster_cap() { return cluster16_ok() ? kMaxSimtCluster : 8; }

int64_t gemm_simt_workspace(const GemmArgs& g) {
  const int s = simt_splits(g);
  return (s > 1 && (s > cluster_cap() || getenv_flag("PFB_SIMT_NO_CLUSTER")))
             ? (int64_t)s * g.batch * g.M * g.N * 4 : 0;
}

template <bool KS>
static void launch_clustered(const GemmArgs& g, dim3 grid, int splits, int64_t kchunk,
                             cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = (unsigned)splits;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  kernel_launches()++;
  cudaLaunchKernelEx(&cfg, gemm_simt_kernel<KS, true>, g, splits, kchunk, (float*)nullptr, false);
}

bool gemm_simt_splittable(const GemmArgs& g) {
  const int64_t tiles = ((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM) * g.batch;
  return g.K > 16 && g.N > 16 && g.K >= 64 && tiles < kNumSMs &&
         (int64_t)g.batch * g.M * g.N < 0x7fffffff;
}

int64_t gemm_simt_workspace_max(const GemmArgs& g) {
  return gemm_simt_splittable(g) ? (int64_t)kSimtWsSplits * g.batch * g.M * g.N * 4 : 0;
}

// splits_want > 0 (autotuner candidates): that many k-splits, reduced over
// DSMEM in one cluster (ws_reduce false, <= cluster limit) or through the
// workspace by a second kernel (ws_reduce true; PFB_E_UNSUPPORTED when the
// workspace is too small)
int gemm_simt_v(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s, int splits_want,
                bool ws_reduce) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return 0;
  if (g.K <= 16) return smallk_launch(g, s);
  // narrow N: warps per row (K split across up to 8 warps for few rows)
  if (g.N <= 16 && !getenv_flag("PFB_SIMT_NO_NARROW"))
    return narrow_launch(g, s);
  int splits = simt_splits(g);
  bool no_cluster = getenv_flag("PFB_SIMT_NO_CLUSTER");
  if (splits_want > 0) {
    if (!gemm_simt_splittable(g)) return PFB_E_UNSUPPORTED;
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(splits_want, g.K / 32));
    if (ws_reduce) {
      if (ws == nullptr || ws_bytes < (int64_t)splits * g.batch * g.M * g.N * 4)
        return PFB_E_UNSUPPORTED;
      no_cluster = true;
    } else {
      splits = std::min(splits, cluster_cap());
    }
  }
  // the workspace path only when clusters cannot hold the splits (or are off)
  bool use_ws = splits > 1 && (no_cluster || splits > cluster_cap());
  if (use_ws && (ws == nullptr || ws_bytes < (int64_t)splits * g.batch * g.M * g.N * 4)) {
    use_ws = false;
    splits = no_cluster ? 1 : std::min(splits, cluster_cap());
  }
  const int64_t kchunk = ((g.K + splits - 1) / splits + BK - 1) / BK * BK;
  splits = (int)((g.K + kchunk - 1) / kchunk);  // no empty splits
  dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM),
            (unsigned)(g.batch * splits));
  if (grid.y > 65535 || grid.z > 65535) return PFB_E_UNSUPPORTED;
  if (splits > 1 && !use_ws) {
    if (g.kscale) launch_clustered<true>(g, grid, splits, kchunk, s);
    else launch_clustered<false>(g, grid, splits, kchunk, s);
    return launch_status();
  }
  float* part = splits > 1 ? (float*)ws : nullptr;
  if (splits > 1 && (int64_t)grid.x * grid.y * (grid.z / splits) > (int64_t)kSimtTiles) {
    // more tiles than tickets: partials, then the reduce kernel
    if (g.kscale)
      launch(gemm_simt_kernel<true, false>, grid, 256, 0, s, g, splits, kchunk, part, false);
    else
      launch(gemm_simt_kernel<false, false>, grid, 256, 0, s, g, splits, kchunk, part, false);
    launch(splitk_reduce, grid_for(g.batch * g.M * g.N, 256), 256, 0, s, g, splits, (const float*)ws);
    return launch_status();
  }
  if (g.kscale)
    launch(gemm_simt_kernel<true, false>, grid, 256, 0, s, g, splits, kchunk, part, true);
  else
    launch(gemm_simt_kernel<false, false>, grid, 256, 0, s, g, splits, kchunk, part, true);
  return launch_status();
}

int gemm_simt(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s) {
  return gemm_simt_v(g, ws, ws_bytes, s, 0, false);
}

}  // namespace pfb
