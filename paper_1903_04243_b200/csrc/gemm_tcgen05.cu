// fp32-accurate GEMM on the 5th-gen tensor cores: tcgen05.mma kind::tf32 with
// a 3xTF32 split, TMA-fed shared-memory pipeline, accumulators in TMEM.
//
//   C = A_hi*B_hi + A_hi*B_lo + A_lo*B_hi,   x_hi = rn_tf32(x), x_lo = rn_tf32(x - x_hi)
// (both exactly representable in TF32, so the tensor core's own operand
// rounding never applies).  Single-pass TF32 misses the fp32 parity bar
// (SURVEY.md §7 "Hard parts"); the dropped terms here are ~2^-22 relative.
//
// Two kernels:
//  1. split_kernel: reads an operand view of any strides through a 32x32
//     shared-memory tile (coalesced on whichever axis is unit-stride) and
//     writes dense K-major hi and lo planes -- so every operand layout
//     (transposed weights, MN-major activations) reaches the tensor core.
//  2. gemm_kernel: persistent (one CTA per SM, static tile stride), 10 warps:
//       warp 0    TMA producer: 4 tiles (A_hi, A_lo, B_hi, B_lo; 32 fp32 of K
//                 = one 128B swizzle row each) per stage, 3-stage ring,
//                 runs ahead across output tiles;
//       warp 1    TMEM allocator + single-thread MMA issuer (UMMA 128x128x8):
//                 4 k-steps x 3 products per stage into one of two TMEM
//                 chunk buffers; every CHUNK_KB stages -> `acc_full[buf]`;
//       warps 2-9 accumulators/epilogue: tcgen05.ld each finished chunk
//                 (warp w owns TMEM lanes 32*(w%4)..+31 and 64 of the 128
//                 columns), add into fp32 registers with round-to-nearest,
//                 release the buffer; after the last chunk of a tile store it
//                 through a conflict-free smem transpose as 4-row x 128-byte
//                 float4 stores (optional per-row scale, accumulate) while the
//                 MMA already fills the next tile.
//     The chunking exists because the tensor core's in-TMEM accumulation
//     truncates: with full-K accumulation the 3xTF32 error grew linearly with
//     K (measured ~1e-4 relative at K=4096); with 64-deep chunks summed in
//     registers it stays at fp32-SIMT level (tests/test_gpu_gemm.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace pfb {
namespace tc {

constexpr int BM = 128, BK = 32, UMMA_K = 8;
#ifndef PFB_CHUNK_KB
#define PFB_CHUNK_KB 2
#endif
constexpr int CHUNK_KB = PFB_CHUNK_KB;            // k-blocks accumulated in TMEM per chunk
constexpr int TILE_BYTES = BM * BK * 4;           // 16 KB per A operand tile
constexpr int kMaxSplit = 8;                      // k-splits per tile (cluster size)
constexpr int EPI_WARPS = 8;                      // split warps; the first DRAIN_WARPS drain
constexpr int EPI_STAGE_FLOATS = 32 * 32;         // per epilogue warp: one 32x32 block,
                                                  // 16B chunks XOR-swizzled by row
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;  // TMA, MMA, 8 split / epilogue warps

// Tile width BN (the MMA's N): 128 (square tiles), 64 or 32 (skinny-M
// problems: more CTAs over N instead of k-splits that must be reduced).
// layout: [stages][epilogue staging, 4 KB per warp, 1 KB aligned for TMA][barriers]
template <int BN_>
struct TileCfg {
  static constexpr int BN = BN_;
  static constexpr int B_BYTES = BN * BK * 4;                 // one B plane per stage
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES + 2 * B_BYTES;  // A_hi, A_lo, B_hi, B_lo
  static constexpr int STAGES = BN == 128 ? 3 : 4;
  // 8 warps x 64 columns (BN 128), 8 x 32 (BN 64), 4 x 32 (BN 32): warp w
  // owns TMEM lanes 32*(w%4)..+31 and DCOLS columns from (w/4)*DCOLS
  static constexpr int DRAIN_WARPS = BN >= 64 ? 8 : 4;
  static constexpr int DCOLS = BN * 4 / DRAIN_WARPS;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                                    EPI_WARPS * EPI_STAGE_FLOATS * 4;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // double-buffered chunks
  // kind::tf32, D=f32, M=128, N=BN; bit 15/16 = A/B MN-major (set per call)
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  static_assert(SMEM_BYTES <= 232448, "shared memory");
};

// ---------------------------------------------------------------------------
// split: x (view [batch, rows, K], any strides) -> dense hi, lo [batch, rows, Kp]

__global__ void __launch_bounds__(256) split_kernel(const float* __restrict__ x, int64_t rows,
                                                    int64_t K, int64_t Kp, int64_t sb, int64_t sr,
                                                    int64_t sk, float* __restrict__ hi,
                                                    float* __restrict__ lo,
                                                    const float* __restrict__ kscale,
                                                    int64_t skb, int64_t skk) {
  pdl_enter();
  __shared__ float t[32][33];
  const int64_t b = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 32;
  const float* xb = x + b * sb;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const bool rows_fast = (sr == 1 && sk != 1);             // MN-major source
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    int64_t r, k;
    if (rows_fast) { r = r0 + tx; k = k0 + ty + j; } else { r = r0 + ty + j; k = k0 + tx; }
    float v = (r < rows && k < K) ? __ldg(xb + r * sr + k * sk) : 0.f;
    if (kscale && k < K) v *= __ldg(kscale + b * skb + k * skk);
    if (rows_fast) t[ty + j][tx] = v; else t[tx][ty + j] = v;  // t[k - k0][r - r0]
  }
  __syncthreads();
  float* hb = hi + b * rows * Kp;
  float* lb = lo + b * rows * Kp;
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    int64_t r = r0 + ty + j, k = k0 + tx;
    if (r < rows && k < Kp) {
      float v = t[tx][ty + j];
      float h = to_tf32(v);
      hb[r * Kp + k] = h;
      lb[r * Kp + k] = tf32_lo(v, h);
    }
  }
}

// Operand feed modes (per operand, chosen on the host):
//   kPreSplit: dense K-major hi/lo planes written by split_kernel (any view)
//   kRawK:     the operand itself, K contiguous -- one TMA box per stage
//   kRawMN:    the operand itself, M/N contiguous -- four 32-wide TMA boxes,
//              consumed by the MMA as an MN-major smem operand
// Raw tiles are split in shared memory by the accumulator warps (hi written
// in place, lo beside it), so small GEMMs need no extra launches.
enum { kPreSplit = 0, kRawK = 1, kRawMN = 2 };

struct Params {
  int M, N, K, batch;
  int ntm, ntn;
  int a_bcast, b_bcast;  // operand shared across the batch
  int a_mode, b_mode;
  uint32_t idesc;
  float* C;
  int64_t scb, scm, scn;
  const float* alpha_rows;
  int accumulate;
  int ksplit;            // >1: a cluster of `ksplit` CTAs per tile, DSMEM reduction
  int kb_per_split;      // k-blocks per split (multiple of CHUNK_KB)
  const float* bias;     // fused epilogue: + bias (broadcast strides), activation
  int64_t sxb, sxm, sxn;
  int act;
  uint32_t mn_lbo, mn_sbo;  // MN-major descriptor strides (4 KB, 512 B)
  int tma_store;            // epilogue stores 32x32 blocks with TMA (map_c)
  unsigned long long* trace;  // PFB_TC_TRACE: globaltimer stamps of CTA 0 (bring-up)
  // second operand pair (C = A B + A2 B2, one accumulation): k-blocks
  // [nk1, nk) come from map_*2 with their own feed modes and broadcast flags
  int nk1;
  int a_mode2, b_mode2, a_bcast2, b_bcast2;
  uint32_t idesc2;
  const float* dy;  // derivative epilogue (GemmArgs::dop)
  int64_t sdb, sdm, sdn;
  int dop;
  int chunk_kb;     // k-blocks accumulated in TMEM per chunk (CHUNK_KB unless overridden)
  int products;     // PFB_TC_PRODUCTS=1: hi*hi only (timing experiments; not fp32-accurate)
  int exp;          // PFB_TC_EXP bits (timing experiments, wrong results): 1 = no TMA after
                    // the first ring fill, 2 = no smem split
};

__device__ __forceinline__ void stamp(const Params& p, int i) {
  if (p.trace != nullptr && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[i] = t;
  }
}

__device__ __forceinline__ void epi4(const Params& p, int bz, int row, int col, float4& v,
                                     const float* bias) {
  if (bias == nullptr && p.act == 0 && p.dop == 0) return;
  float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (bias && col + j < p.N)
      e[j] += __ldg(bias + (int64_t)bz * p.sxb + (int64_t)row * p.sxm + (int64_t)(col + j) * p.sxn);
    e[j] = apply_act(p.act, e[j]);
    if (p.dop && col + j < p.N)
      e[j] *= dop_factor(p.dop, p.dy,
                         (int64_t)bz * p.sdb + (int64_t)row * p.sdm + (int64_t)(col + j) * p.sdn);
  }
  v = make_float4(e[0], e[1], e[2], e[3]);
}

// epilogue operands of 4 consecutive columns, loaded ahead of use (the
// loads of a whole block are issued before the first is consumed: one
// memory round trip per block instead of one per element)
struct Epi4 {
  float b[4], y[4];
};

__device__ __forceinline__ void epi4_load(const Params& p, const float* bias, int bz, int row,
                                          int col, Epi4& e) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool ok = col + j < p.N;
    e.b[j] = (bias && ok) ? __ldg(bias + (int64_t)bz * p.sxb + (int64_t)row * p.sxm +
                                  (int64_t)(col + j) * p.sxn) : 0.f;
    e.y[j] = (p.dop && ok) ? __ldg(p.dy + (int64_t)bz * p.sdb + (int64_t)row * p.sdm +
                                   (int64_t)(col + j) * p.sdn) : 0.f;
  }
}

__device__ __forceinline__ void epi4_apply(const Params& p, const Epi4& e, float4& v) {
  float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    x[j] = apply_act(p.act, x[j] + e.b[j]);
    if (p.dop) x[j] *= p.dop == PFB_DOP_DTANH ? 1.f - e.y[j] * e.y[j] : e.y[j] * (1.f - e.y[j]);
  }
  v = make_float4(x[0], x[1], x[2], x[3]);
}

__device__ __forceinline__ void tma_load_operand(const CUtensorMap* mh, const CUtensorMap* ml,
                                                 int mode, uint64_t* bar, uint8_t* dst_hi,
                                                 uint8_t* dst_lo, int kb, int row0, int z,
                                                 int rows) {
  if (mode == kRawMN) {
    for (int j = 0; j < rows / 32; ++j) tma_load_3d(mh, bar, dst_hi + j * 4096, row0 + 32 * j, kb * BK, z);
  } else {
    tma_load_3d(mh, bar, dst_hi, kb * BK, row0, z);
    if (mode == kPreSplit) tma_load_3d(ml, bar, dst_lo, kb * BK, row0, z);
  }
}

// raw tiles split in place (tc_ptx.cuh), 256 split threads
__device__ __forceinline__ void split_tile_smem(uint8_t* hi, uint8_t* lo, int bytes, int t) {
  split_tf32_smem(smem_u32(hi), smem_u32(lo), bytes / 16, t, 32 * EPI_WARPS);
}

// Rows [rb, re) of the split-K tile summed over the cluster's KS partial
// tiles (each CTA's own smem, rows x BN floats, 16-byte chunks XOR-swizzled by
// row), in rank order -> the epilogue -> C.  Up to 16 remote 16-byte loads are
// issued before the first is added (DSMEM latency ~200 cycles each).
__device__ __forceinline__ float4 ld_dsmem_f4_nv(uint32_t remote) {
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(remote));
  return v;
}

template <int KS, int BN>
__device__ __forceinline__ void cluster_reduce(const Params& p, uint32_t red, int rb, int re,
                                               int m0, int n0, int bz) {
  constexpr int PER = 16 / KS;  // items per pass per thread
  uint32_t base[KS];
#pragma unroll
  for (int q = 0; q < KS; ++q)
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(base[q]) : "r"(red), "r"(q));
  const int items = (re - rb) * (BN / 4);
  float* cbase = p.C + bz * p.scb;
  const float* rbias = p.alpha_rows != nullptr ? p.bias : nullptr;  // else in split 0's partial
  const bool has_epi = rbias != nullptr || p.act != 0 || p.dop != 0;
  for (int i0 = threadIdx.x; i0 < items; i0 += PER * NUM_THREADS) {
    float4 w[PER][KS];
    Epi4 ep[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = i0 + j * NUM_THREADS;
      if (idx < items) {
        const int row = rb + idx / (BN / 4), ch = idx % (BN / 4);
        const uint32_t off = (uint32_t)(row * BN + 4 * (ch ^ (row & 7))) * 4u;
#pragma unroll
        for (int q = 0; q < KS; ++q) w[j][q] = ld_dsmem_f4_nv(base[q] + off);
        if (has_epi && m0 + row < p.M) epi4_load(p, rbias, bz, m0 + row, n0 + 4 * ch, ep[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = i0 + j * NUM_THREADS;
      if (idx >= items) continue;
      float4 v = w[j][0];
#pragma unroll
      for (int q = 1; q < KS; ++q) { v.x += w[j][q].x; v.y += w[j][q].y; v.z += w[j][q].z; v.w += w[j][q].w; }
      const int row = rb + idx / (BN / 4), ch = idx % (BN / 4);
      const int grow = m0 + row, col = n0 + 4 * ch;
      if (grow >= p.M) continue;
      const float alpha = p.alpha_rows ? __ldg(p.alpha_rows + (int64_t)bz * p.M + grow) : 1.f;
      v.x *= alpha; v.y *= alpha; v.z *= alpha; v.w *= alpha;
      float* q = cbase + (int64_t)grow * p.scm + (int64_t)col * p.scn;
      if (p.scn == 1 && col + 3 < p.N && ((reinterpret_cast<uintptr_t>(q) & 15) == 0)) {
        if (p.accumulate) {
          const float4 o = *reinterpret_cast<const float4*>(q);
          v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        }
        if (has_epi) epi4_apply(p, ep[j], v);
        *reinterpret_cast<float4*>(q) = v;
      } else {
        if (p.accumulate) {
          if (col < p.N) v.x += q[0];
          if (col + 1 < p.N) v.y += q[p.scn];
          if (col + 2 < p.N) v.z += q[2 * p.scn];
          if (col + 3 < p.N) v.w += q[3 * p.scn];
        }
        if (has_epi) epi4_apply(p, ep[j], v);
        const float e[4] = {v.x, v.y, v.z, v.w};
        for (int jj = 0; jj < 4; ++jj)
          if (col + jj < p.N) q[(int64_t)jj * p.scn] = e[jj];
      }
    }
  }
}

template <int BN_>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_ah, const __grid_constant__ CUtensorMap map_al,
            const __grid_constant__ CUtensorMap map_bh, const __grid_constant__ CUtensorMap map_bl,
            const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_ah2,
            const __grid_constant__ CUtensorMap map_al2, const __grid_constant__ CUtensorMap map_bh2,
            const __grid_constant__ CUtensorMap map_bl2, Params p) {
  using C = TileCfg<BN_>;
  constexpr int BN = C::BN, STAGES = C::STAGES, STAGE_BYTES = C::STAGE_BYTES;
  constexpr int DCOLS = C::DCOLS, DRAIN_WARPS = C::DRAIN_WARPS;
  stamp(p, 0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES +
                                               EPI_WARPS * EPI_STAGE_FLOATS * 4);
  uint64_t* full = bars;                   // [STAGES] TMA -> (split) -> MMA
  uint64_t* empty = bars + STAGES;         // [STAGES] MMA -> TMA
  uint64_t* ready = bars + 2 * STAGES;     // [STAGES] smem split -> MMA
  uint64_t* acc_full = bars + 3 * STAGES;  // [2] MMA -> accumulators
  uint64_t* acc_empty = acc_full + 2;      // [2] accumulators -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (p.K + BK - 1) / BK;
  const int tiles_per_batch = p.ntm * p.ntn;
  const bool clustered = p.ksplit > 1;
  // clustered: exactly one work unit per CTA (cluster rank = k-split index)
  const int ntiles = clustered ? (int)blockIdx.x + 1 : tiles_per_batch * p.batch * p.ksplit;
  const int ustride = clustered ? 1 : (int)gridDim.x;
  const bool dual = p.nk1 < (p.K + BK - 1) / BK;
  const bool split_smem = p.a_mode != kPreSplit || p.b_mode != kPreSplit ||
                          (dual && (p.a_mode2 != kPreSplit || p.b_mode2 != kPreSplit));

  auto tile = [&](int s, int which) {
    return smem + s * STAGE_BYTES + (which < 2 ? which * TILE_BYTES
                                               : 2 * TILE_BYTES + (which - 2) * C::B_BYTES);
  };
  // which: 0 = A_hi, 1 = A_lo, 2 = B_hi, 3 = B_lo

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], EPI_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 32 * DRAIN_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ah)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_al)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bl)) : "memory");
    if (dual) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ah2)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bh2)) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;
  // the prologue above (barriers, TMEM, descriptor prefetch) overlaps the
  // previous kernel's tail under programmatic dependent launch; operands are
  // only read after this wait
  if (threadIdx.x == 0) stamp(p, 1);
  pdl_enter();
  if (threadIdx.x == 0) stamp(p, 2);
  if (threadIdx.x == 0 && p.trace != nullptr && blockIdx.x < 160) {  // per-CTA start
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[192 + blockIdx.x] = t;
  }

  auto a_bytes = [&](int mode) { return (mode == kPreSplit ? 2 : 1) * TILE_BYTES; };
  auto b_bytes = [&](int mode) { return (mode == kPreSplit ? 2 : 1) * C::B_BYTES; };

  if (warp == 0) {
    if (lane == 0 && !(p.exp & 32)) {
      int g = 0;
      for (int u = blockIdx.x; u < ntiles; u += ustride) {
        const int t = u / p.ksplit, ks = u % p.ksplit;
        const int bz = t / tiles_per_batch, r = t % tiles_per_batch;
        const int m0 = (r / p.ntn) * BM, n0 = (r % p.ntn) * BN;
        const int kb0 = ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
          if (g < 16) stamp(p, 80 + g);
          if ((p.exp & 1) && g >= STAGES) {
            mbar_arrive(&full[s]);  // experiment: stages reused without reloading
          } else if (kb < p.nk1) {
            const int za = p.a_bcast ? 0 : bz, zb = p.b_bcast ? 0 : bz;
            if (g < 16) stamp(p, 16 + g);
            mbar_expect_tx(&full[s], a_bytes(p.a_mode) + b_bytes(p.b_mode));
            tma_load_operand(&map_ah, &map_al, p.a_mode, &full[s], tile(s, 0), tile(s, 1), kb, m0, za, BM);
            tma_load_operand(&map_bh, &map_bl, p.b_mode, &full[s], tile(s, 2), tile(s, 3), kb, n0, zb, BN);
          } else {
            const int za = p.a_bcast2 ? 0 : bz, zb = p.b_bcast2 ? 0 : bz, k2 = kb - p.nk1;
            mbar_expect_tx(&full[s], a_bytes(p.a_mode2) + b_bytes(p.b_mode2));
            tma_load_operand(&map_ah2, &map_al2, p.a_mode2, &full[s], tile(s, 0), tile(s, 1), k2, m0, za, BM);
            tma_load_operand(&map_bh2, &map_bl2, p.b_mode2, &full[s], tile(s, 2), tile(s, 3), k2, n0, zb, BN);
          }
          if (g == 0) stamp(p, 3);
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the loop (warp-uniform control flow: descriptors
    // and TMEM addresses stay in uniform registers); one elected lane issues
    // each k-block's MMAs and commits
    int g = 0, gc = 0;
    for (int u = blockIdx.x; u < ntiles; u += ustride) {
      const int ks = u % p.ksplit;
      const int kb0 = ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
      const int uchunks = (kb1 - kb0 + p.chunk_kb - 1) / p.chunk_kb;
      for (int c = 0; c < uchunks; ++c, ++gc) {
        const int buf = gc & 1;
        if (gc >= 2 && !(p.exp & 4)) mbar_wait(&acc_empty[buf], ((gc >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t tmem_d = tmem_base + (uint32_t)(buf * BN);
        const int kb_beg = kb0 + c * p.chunk_kb;
        const int kb_end = min(kb1, kb_beg + p.chunk_kb);
        for (int kb = kb_beg; kb < kb_end; ++kb, ++g) {
          const int s = g % STAGES;
          if (!(p.exp & 16)) mbar_wait(split_smem ? &ready[s] : &full[s], (g / STAGES) & 1);
          if (lane == 0) {
            if (g == 0) stamp(p, 5);
            if (g < 16) stamp(p, 64 + g);
            if (g < 16 && p.trace != nullptr && blockIdx.x == 0) p.trace[96 + g] = clock64();
          }
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t a0 = smem_u32(tile(s, 0)), a1 = smem_u32(tile(s, 1));
          const uint32_t b0 = smem_u32(tile(s, 2)), b1 = smem_u32(tile(s, 3));
          const bool second = kb >= p.nk1;
          const int am_ = second ? p.a_mode2 : p.a_mode, bm_ = second ? p.b_mode2 : p.b_mode;
          const uint32_t idesc = second ? p.idesc2 : p.idesc;
          const bool amn = am_ == kRawMN, bmn = bm_ == kRawMN;
          const uint64_t a_hi = amn ? smem_desc_mn_sw128(a0, p.mn_lbo, p.mn_sbo) : smem_desc_sw128(a0);
          const uint64_t a_lo = amn ? smem_desc_mn_sw128(a1, p.mn_lbo, p.mn_sbo) : smem_desc_sw128(a1);
          const uint64_t b_hi = bmn ? smem_desc_mn_sw128(b0, p.mn_lbo, p.mn_sbo) : smem_desc_sw128(b0);
          const uint64_t b_lo = bmn ? smem_desc_mn_sw128(b1, p.mn_lbo, p.mn_sbo) : smem_desc_sw128(b1);
          // k-step advance: +32 B inside the swizzle row (K-major) or one
          // 1 KB atom (MN-major)
          const uint64_t astep = amn ? (1024 >> 4) : ((UMMA_K * 4) >> 4);
          const uint64_t bstep = bmn ? (1024 >> 4) : ((UMMA_K * 4) >> 4);
          const bool lo_lo = am_ != kPreSplit && bm_ != kPreSplit;
          const bool three = p.products != 1;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t da = astep * k, db = bstep * k;
              const uint32_t acc = (kb > kb_beg || k > 0) ? 1u : 0u;
              mma_tf32(tmem_d, a_hi + da, b_hi + db, idesc, acc);
              if (three) {
                mma_tf32(tmem_d, a_hi + da, b_lo + db, idesc, 1u);
                mma_tf32(tmem_d, a_lo + da, b_hi + db, idesc, 1u);
                // both operands raw: hi = trunc_tf32 on both sides makes the
                // dropped lo*lo term sign-biased, so it is kept
                if (lo_lo) mma_tf32(tmem_d, a_lo + da, b_lo + db, idesc, 1u);
              }
            }
            mma_commit(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(&acc_full[buf]);
        __syncwarp();
      }
    }
    if (lane == 0) stamp(p, 6);
    __syncwarp();
  } else {
    // ---- split + accumulators + epilogue (warps 2..9): warp w owns TMEM
    // lanes 32*(w%4)..+31 (its rows) and columns [half*64, half*64+64) ----
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;  // 0..255
    float* stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES) +
                   (warp - 2) * EPI_STAGE_FLOATS;
    int gc = 0, gs = 0;
    auto split_stage = [&](int kb) {
      const int s = gs % STAGES;
      mbar_wait(&full[s], (gs / STAGES) & 1);
      if (gs == 0 && et == 0) stamp(p, 4);
      if (gs < 16 && et == 0) stamp(p, 32 + gs);
      const bool second = kb >= p.nk1;
      if ((second ? p.a_mode2 : p.a_mode) != kPreSplit && !(p.exp & 2))
        split_tile_smem(tile(s, 0), tile(s, 1), TILE_BYTES, et);
      if ((second ? p.b_mode2 : p.b_mode) != kPreSplit && !(p.exp & 2))
        split_tile_smem(tile(s, 2), tile(s, 3), C::B_BYTES, et);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
      if (gs < 16 && et == 0) stamp(p, 48 + gs);
      ++gs;
    };
    float acc[DCOLS];
    const bool drains = (warp - 2) < DRAIN_WARPS;
    auto drain = [&]() {
      const int buf = gc & 1;
      ++gc;
      if (!drains || (p.exp & 4)) return;
      mbar_wait(&acc_full[buf], ((gc - 1) >> 1) & 1);
      if (gc == 1 && et == 0) stamp(p, 7);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int cc = 0; cc < DCOLS; cc += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) +
                      (uint32_t)(buf * BN + half * DCOLS + cc), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[cc + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&acc_empty[buf]);
    };
    for (int u = blockIdx.x; u < ntiles; u += ustride) {
      const int t = u / p.ksplit, ks = u % p.ksplit;
      const int bz = t / tiles_per_batch, r = t % tiles_per_batch;
      const int m0 = (r / p.ntn) * BM, n0 = (r % p.ntn) * BN;
      const int kb0 = ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
      const int uchunks = (kb1 - kb0 + p.chunk_kb - 1) / p.chunk_kb;
      // the bias starts the accumulation of split 0 (its loads overlap the
      // k-loop instead of stalling the epilogue); a row scale must not scale it
      const float* abias = (ks == 0 && p.alpha_rows == nullptr) ? p.bias : nullptr;
      if (abias != nullptr && drains) {
        const int grow = m0 + quarter * 32 + lane;
        const int64_t rb = (int64_t)bz * p.sxb + (int64_t)grow * p.sxm;
#pragma unroll
        for (int j = 0; j < DCOLS; ++j) {
          const int col = n0 + half * DCOLS + j;
          acc[j] = (grow < p.M && col < p.N) ? __ldg(abias + rb + (int64_t)col * p.sxn) : 0.f;
        }
      } else {
#pragma unroll
        for (int j = 0; j < DCOLS; ++j) acc[j] = 0.f;
      }
      // split chunk c's stages, then drain chunk c-1 (the MMA works on
      // chunk c-1 while the stages of chunk c are being split)
      for (int c = 0; c < uchunks; ++c) {
        if (split_smem) {
          const int kb_beg = kb0 + c * p.chunk_kb, kb_end = min(kb1, kb_beg + p.chunk_kb);
          if (!(p.exp & 32))
            for (int kb = kb_beg; kb < kb_end; ++kb) split_stage(kb);
        }
        if (c > 0) drain();
      }
      drain();
      if (!drains) continue;
      // bias: folded into split 0's accumulator above unless rows are scaled
      const float* ubias = (p.alpha_rows != nullptr && ks == 0) ? p.bias : nullptr;
      if (clustered) {
        // partial tile -> own smem (stage area is idle: every MMA of this
        // CTA's only unit has completed), rows x BN/4 float4, XOR-swizzled
        float* red = reinterpret_cast<float*>(smem);
        const int row = quarter * 32 + lane;
#pragma unroll
        for (int j = 0; j < DCOLS / 4; ++j) {
          const int ch = half * (DCOLS / 4) + j;
          *reinterpret_cast<float4*>(red + row * BN + 4 * (ch ^ (row & 7))) =
              make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
        }
        continue;
      }
      const int row0 = m0 + quarter * 32;
      if (p.tma_store) {
        // the staging block's XOR layout is TMA's SWIZZLE_128B: write the
        // finished 32x32 block, one bulk tensor store per block (bounds
        // clipped by the map), staging reuse gated on the bulk read
        const int grow = row0 + lane;
        const float alpha =
            (p.alpha_rows && grow < p.M) ? __ldg(p.alpha_rows + (int64_t)bz * p.M + grow) : 1.f;
        const bool epi = (ubias != nullptr || p.act != 0 || p.dop != 0) && grow < p.M;
#pragma unroll
        for (int cc = 0; cc < DCOLS; cc += 32) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
          const int col0 = n0 + half * DCOLS + cc;
#pragma unroll
          for (int h = 0; h < 8; h += 4) {
            Epi4 e[4];
            if (epi) {
#pragma unroll
              for (int q = 0; q < 4; ++q) epi4_load(p, ubias, bz, grow, col0 + 4 * (h + q), e[q]);
            }
#pragma unroll
            for (int q = h; q < h + 4; ++q) {
              float4 v = make_float4(acc[cc + 4 * q] * alpha, acc[cc + 4 * q + 1] * alpha,
                                     acc[cc + 4 * q + 2] * alpha, acc[cc + 4 * q + 3] * alpha);
              if (epi) epi4_apply(p, e[q - h], v);
              *reinterpret_cast<float4*>(stage + lane * 32 + 4 * (q ^ (lane & 7))) = v;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&map_c, stage, col0, row0, bz);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        continue;
      }
      // 32x32 blocks through smem: each lane writes its row as float4s, then
      // every store instruction covers 4 rows x 128 contiguous bytes
      float* cbase = p.C + bz * p.scb;
      const int64_t ldm = p.scm, ldn = p.scn;
      const int sub_r = lane >> 3, sub_c = (lane & 7) * 4;
#pragma unroll
      for (int cc = 0; cc < DCOLS; cc += 32) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stage + lane * 32 + 4 * (q ^ (lane & 7))) =
              make_float4(acc[cc + 4 * q], acc[cc + 4 * q + 1], acc[cc + 4 * q + 2],
                          acc[cc + 4 * q + 3]);
        __syncwarp();
        const int col = n0 + half * DCOLS + cc + sub_c;
#pragma unroll 4
        for (int i = 0; i < 32; i += 4) {
          const int row = row0 + i + sub_r;
          if (row < p.M) {
            const float alpha = p.alpha_rows ? __ldg(p.alpha_rows + (int64_t)bz * p.M + row) : 1.f;
            const int srow = i + sub_r;
            float4 v = *reinterpret_cast<const float4*>(
                stage + srow * 32 + 4 * ((sub_c >> 2) ^ (srow & 7)));
            v.x *= alpha; v.y *= alpha; v.z *= alpha; v.w *= alpha;
            float* q = cbase + (int64_t)row * ldm + (int64_t)col * ldn;
            if (ldn == 1 && col + 3 < p.N && ((reinterpret_cast<uintptr_t>(q) & 15) == 0)) {
              if (p.accumulate) {
                const float4 o = *reinterpret_cast<const float4*>(q);
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              epi4(p, bz, row, col, v, ubias);
              *reinterpret_cast<float4*>(q) = v;
            } else {
              if (p.accumulate) {
                const float* qq = q;
                if (col < p.N) v.x += qq[0];
                if (col + 1 < p.N) v.y += qq[ldn];
                if (col + 2 < p.N) v.z += qq[2 * ldn];
                if (col + 3 < p.N) v.w += qq[3 * ldn];
              }
              epi4(p, bz, row, col, v, ubias);
              const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (col + j < p.N) q[(int64_t)j * ldn] = e[j];
            }
          }
        }
        __syncwarp();
      }
    }
  }
  if (threadIdx.x == 64) stamp(p, 8);
  if (p.tma_store && warp >= 2 && lane == 0)
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) stamp(p, 9);
  if (clustered) {
    // deterministic split-K reduction over DSMEM: CTA `rank` of the cluster
    // sums rows [rank*rows_per, ...) of all partial tiles in rank order
    cluster_sync_all();
    const int t = blockIdx.x / p.ksplit;
    const int bz = t / tiles_per_batch, r = t % tiles_per_batch;
    const int m0 = (r / p.ntn) * BM, n0 = (r % p.ntn) * BN;
    const int rank = (int)cluster_rank();
    const int rows_per = (BM + p.ksplit - 1) / p.ksplit;
    const int rb = rank * rows_per, re = min(BM, rb + rows_per);
    const uint32_t red = smem_u32(smem);
    switch (p.ksplit) {
      case 2: cluster_reduce<2, BN>(p, red, rb, re, m0, n0, bz); break;
      case 3: cluster_reduce<3, BN>(p, red, rb, re, m0, n0, bz); break;
      case 4: cluster_reduce<4, BN>(p, red, rb, re, m0, n0, bz); break;
      case 5: cluster_reduce<5, BN>(p, red, rb, re, m0, n0, bz); break;
      case 6: cluster_reduce<6, BN>(p, red, rb, re, m0, n0, bz); break;
      case 7: cluster_reduce<7, BN>(p, red, rb, re, m0, n0, bz); break;
      default: cluster_reduce<8, BN>(p, red, rb, re, m0, n0, bz); break;
    }
    cluster_sync_all();  // peers' smem stays live until every CTA has read it
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
    if (lane == 0) stamp(p, 10);
    if (lane == 0 && p.trace != nullptr && blockIdx.x < 160) {  // per-CTA end
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[352 + blockIdx.x] = t;
    }
  }
}

// --- host side -------------------------------------------------------------

// dense K-major plane [batch][rows][Kp]
static bool make_map(CUtensorMap* map, const float* base, int64_t Kp, int64_t rows, int64_t batch,
                     int box_rows = BM) {
  cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(Kp * 4), (cuuint64_t)(rows * Kp * 4)};
  cuuint32_t box[3] = {BK, (cuuint32_t)box_rows, 1};
  return encode(map, base, dims, strides, box);
}

// Can the operand view (rows x K per batch, strides in elements) be read by
// TMA directly?  Returns kRawK / kRawMN, or kPreSplit when it cannot.
static int raw_mode(const float* base, int64_t rows, int64_t K, int64_t nb, int64_t sb, int64_t sr,
                    int64_t sk) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return kPreSplit;
  const bool b_ok = nb == 1 || ((sb * 4) % 16 == 0 && sb > 0);
  if (!b_ok) return kPreSplit;
  if (sk == 1 && (rows == 1 || ((sr * 4) % 16 == 0 && sr >= K))) return kRawK;
  if (sr == 1 && rows > 1 && (sk * 4) % 16 == 0 && sk >= rows) return kRawMN;
  return kPreSplit;
}

static bool make_raw_map(CUtensorMap* map, int mode, const float* base, int64_t rows, int64_t K,
                         int64_t nb, int64_t sb, int64_t sr, int64_t sk, int box_rows = BM) {
  if (mode == kRawK) {
    const int64_t ld = rows == 1 ? (K + 3) / 4 * 4 : sr;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)nb};
    cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)((nb == 1 ? ld * rows : sb) * 4)};
    cuuint32_t box[3] = {BK, (cuuint32_t)box_rows, 1};
    return encode(map, base, dims, strides, box);
  }
  cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)K, (cuuint64_t)nb};
  cuuint64_t strides[2] = {(cuuint64_t)(sk * 4), (cuuint64_t)((nb == 1 ? sk * K : sb) * 4)};
  cuuint32_t box[3] = {32, BK, 1};
  return encode(map, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = kNumSMs;
  }
  return n;
}

static int64_t align_up(int64_t x) { return (x + 255) / 256 * 256; }

// K-splits so that (tiles x splits) covers the SMs, >= 2 chunks per split;
// the splits of one tile form a thread-block cluster (<= 8, portable size)
constexpr int kMaxCluster = kMaxSplit;
static int chunk_kb() {
  static const int c = [] {
    const char* e = getenv("PFB_TC_CHUNK");
    const int v = e ? atoi(e) : CHUNK_KB;
    return v >= 1 && v <= 16 ? v : CHUNK_KB;
  }();
  return c;
}

static void choose_split(const GemmArgs& g, int* ksplit, int* kb_per, int BN = 128) {
  const int CHUNK_KB = chunk_kb();
  const int64_t tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN) * g.batch;
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int nk = (int)((Kp + BK - 1) / BK);
  // time model (us): waves x (k-blocks per unit x 0.6 + 1.5), +4 for the reduction
  auto cost = [&](int s, int* per_out) {
    int per = (nk + s - 1) / s;
    per = (per + CHUNK_KB - 1) / CHUNK_KB * CHUNK_KB;
    const int real = (nk + per - 1) / per;
    *per_out = per;
    const double waves = std::ceil((double)tiles * real / num_sms());
    return waves * (per * 0.6 + 1.5) + (real > 1 ? 1.0 : 0.0);
  };
  int best_per = 0;
  double best = cost(1, &best_per);
  int s_max = 1;
  if (tiles < num_sms() && nk >= 4 * CHUNK_KB)
    s_max = (int)std::max<int64_t>(1, std::min<int64_t>(
        std::min<int64_t>((num_sms() + tiles - 1) / tiles, nk / (2 * CHUNK_KB)), kMaxCluster));
  for (int s = 2; s <= s_max; ++s) {
    int per;
    const double c = cost(s, &per);
    if (c < best) { best = c; best_per = per; }
  }
  *kb_per = best_per;
  *ksplit = (nk + best_per - 1) / best_per;
}

}  // namespace tc

void tc_split_launch(const float* x, int64_t batch, int64_t rows, int64_t K, int64_t Kp, int64_t sb,
                     int64_t sr, int64_t sk, float* hi, float* lo, const float* kscale,
                     int64_t skb, int64_t skk, cudaStream_t s) {
  dim3 grid((unsigned)((Kp + 31) / 32), (unsigned)((rows + 31) / 32), (unsigned)batch);
  launch(tc::split_kernel, grid, 256, 0, s, x, rows, K, Kp, sb, sr, sk, hi, lo, kscale, skb, skk);
}

// PFB_TC_TRACE=1: CTA 0 of every tcgen05 GEMM launch writes globaltimer
// stamps (entry, after PDL wait, after prologue, first TMA issued, first
// stage landed, first MMA issued, last commit, first accumulator ready,
// epilogue done, CTA done, TMEM freed) -- read with pfb_debug_tc_trace().
static unsigned long long* g_trace = nullptr;
unsigned long long* tc_trace_buffer() {
  static const bool on = getenv_flag("PFB_TC_TRACE");
  if (on && g_trace == nullptr) {
    cudaMalloc(&g_trace, 512 * sizeof(unsigned long long));
    cudaMemset(g_trace, 0, 512 * sizeof(unsigned long long));
  }
  return on ? g_trace : nullptr;
}

// Workspace: hi/lo planes of both operands for the pre-split feed (K padded
// to a multiple of 4 so every TMA row stride is 16-byte aligned); raw-fed
// operands use none of it.
int64_t gemm_tcgen05_workspace(const GemmArgs& g) {
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int64_t ba = (g.sab == 0 && g.batch > 1) ? 1 : g.batch;
  const int64_t bb = (g.sbb == 0 && g.batch > 1) ? 1 : g.batch;
  return 2 * tc::align_up(ba * g.M * Kp * 4) + 2 * tc::align_up(bb * g.N * Kp * 4);
}

int64_t gemm_planes_bytes(const GemmArgs& g) {
  if (g.kscale) return 0;
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int64_t bb = (g.sbb == 0 && g.batch > 1) ? 1 : g.batch;
  return 2 * tc::align_up(bb * g.N * Kp * 4);
}

bool gemm_tcgen05_eligible(const GemmArgs& g) {
  if (g.K < 8 || g.M < 1 || g.N < 8) return false;
  return !(g.M > (1ll << 31) || g.N > (1ll << 31) || g.K > (1ll << 31) || g.batch > 65535 ||
           (g.M + 31) / 32 > 65535 || (g.N + 31) / 32 > 65535);
}

// Does the raw (in-smem split) feed apply to at least one operand?
bool gemm_tcgen05_raw_possible(const GemmArgs& g) {
  using namespace tc;
  const int64_t ba = (g.sab == 0 && g.batch > 1) ? 1 : g.batch;
  const int64_t bb = (g.sbb == 0 && g.batch > 1) ? 1 : g.batch;
  return raw_mode(g.A, g.M, g.K, ba, g.sab, g.sam, g.sak) != kPreSplit ||
         raw_mode(g.B, g.N, g.K, bb, g.sbb, g.sbn, g.sbk) != kPreSplit;
}

// Dispatch model (microseconds), calibrated on B200 (tools/gemm_probe.py):
// tensor path ~0.6 us per 32-deep k-block per 128x128 tile per wave plus
// fixed launch costs; SIMT fp32 ~15 TFLOP/s.  Skinny problems with few
// tiles (batch-128 forward passes) go SIMT with split-K.
bool gemm_tcgen05_profitable(const GemmArgs& g) {
  if (g.K < 16 || g.M < 16 || g.N < 16) return false;
  const double tiles = (double)((g.M + 127) / 128) * ((g.N + 127) / 128) * g.batch;
  int ks, per;
  tc::choose_split(g, &ks, &per);
  const double nk = (double)per;
  const double waves = std::ceil(tiles * ks / tc::num_sms());
  const double t_tc = waves * (nk * 0.6 + 1.5) + 3.0 + (ks > 1 ? 1.0 : 0.0);
  const double t_simt = 2.0 * g.M * g.N * g.K * g.batch / 15e6 + 3.0;
  return t_tc < t_simt;
}

// variant: 0 = auto (raw feed for small problems), 1 = pre-split both
// operands, 2 = raw feed wherever the operand layout allows it
namespace tc {

// One operand pair's TMA feed: raw maps (split in smem) or pre-split hi/lo
// planes written into the workspace at `w` (advanced past what it uses).
struct PairFeed {
  CUtensorMap ah, al, bh, bl;
  int am = kPreSplit, bm = kPreSplit, a_bc = 0, b_bc = 0;
  int64_t Kp = 0;
};

static int64_t pair_need(const GemmArgs& g, int variant, int* am_out, int* bm_out) {
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int a_bc = g.sab == 0 && g.batch > 1;
  const int b_bc = g.sbb == 0 && g.batch > 1 && !(g.kscale && g.skb != 0);
  const int64_t ba = a_bc ? 1 : g.batch, bb = b_bc ? 1 : g.batch;
  int am = kPreSplit, bm = kPreSplit;
  if (variant == 2 || variant == 3)  // 3: A raw, B pre-split
    am = raw_mode(g.A, g.M, g.K, ba, g.sab, g.sam, g.sak);
  if ((variant == 2 || variant == 4) && !g.b_hi)  // 4: A pre-split, B raw
    bm = g.kscale ? kPreSplit : raw_mode(g.B, g.N, g.K, bb, g.sbb, g.sbn, g.sbk);
  *am_out = am;
  *bm_out = bm;
  return (am == kPreSplit ? 2 * align_up(ba * g.M * Kp * 4) : 0) +
         (bm == kPreSplit && !g.b_hi ? 2 * align_up(bb * g.N * Kp * 4) : 0);
}

static int prep_pair(const GemmArgs& g, int variant, char*& w, cudaStream_t s, PairFeed* f,
                     int bn = 128) {
  f->Kp = (g.K + 3) / 4 * 4;
  const int64_t Kp = f->Kp;
  // a per-batch kscale makes B's planes differ per batch even for a shared B
  f->a_bc = g.sab == 0 && g.batch > 1;
  f->b_bc = g.sbb == 0 && g.batch > 1 && !(g.kscale && g.skb != 0);
  const int64_t ba = f->a_bc ? 1 : g.batch, bb = f->b_bc ? 1 : g.batch;
  pair_need(g, variant, &f->am, &f->bm);
  if (f->am == kPreSplit) {
    float* ah = reinterpret_cast<float*>(w); w += align_up(ba * g.M * Kp * 4);
    float* al = reinterpret_cast<float*>(w); w += align_up(ba * g.M * Kp * 4);
    dim3 ga((unsigned)((Kp + 31) / 32), (unsigned)((g.M + 31) / 32), (unsigned)ba);
    launch(split_kernel, ga, 256, 0, s, g.A, g.M, g.K, Kp, g.sab, g.sam, g.sak, ah, al,
           (const float*)nullptr, (int64_t)0, (int64_t)0);
    if (!make_map(&f->ah, ah, Kp, g.M, ba) || !make_map(&f->al, al, Kp, g.M, ba)) return PFB_E_UNSUPPORTED;
  } else {
    if (!make_raw_map(&f->ah, f->am, g.A, g.M, g.K, ba, g.sab, g.sam, g.sak)) return PFB_E_UNSUPPORTED;
    f->al = f->ah;
  }
  if (f->bm == kRawMN && bn % 32 != 0) f->bm = kPreSplit;
  if (f->bm == kPreSplit && g.b_hi) {  // planes made once by pfb_gemm_split_planes
    if (!make_map(&f->bh, g.b_hi, Kp, g.N, bb, bn) || !make_map(&f->bl, g.b_lo, Kp, g.N, bb, bn))
      return PFB_E_UNSUPPORTED;
  } else if (f->bm == kPreSplit) {
    float* bh = reinterpret_cast<float*>(w); w += align_up(bb * g.N * Kp * 4);
    float* bl = reinterpret_cast<float*>(w); w += align_up(bb * g.N * Kp * 4);
    dim3 gb((unsigned)((Kp + 31) / 32), (unsigned)((g.N + 31) / 32), (unsigned)bb);
    launch(split_kernel, gb, 256, 0, s, g.B, g.N, g.K, Kp, g.sbb, g.sbn, g.sbk, bh, bl, g.kscale,
           g.skb, g.skk);
    if (!make_map(&f->bh, bh, Kp, g.N, bb, bn) || !make_map(&f->bl, bl, Kp, g.N, bb, bn))
      return PFB_E_UNSUPPORTED;
  } else {
    if (!make_raw_map(&f->bh, f->bm, g.B, g.N, g.K, bb, g.sbb, g.sbn, g.sbk, bn))
      return PFB_E_UNSUPPORTED;
    f->bl = f->bh;
  }
  return 0;
}

// g carries the output, epilogue and (for the split model) the total K;
// f2 == nullptr: one operand pair
template <int BN>
static int launch_gemm(const GemmArgs& g, const PairFeed& f1, const PairFeed* f2, cudaStream_t s,
                       int ksplit_want) {
  using C = TileCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM_BYTES);
    attr = true;
  }
  const int nk1 = (int)((f1.Kp + BK - 1) / BK);
  const int nk = nk1 + (f2 ? (int)((f2->Kp + BK - 1) / BK) : 0);
  GemmArgs gm = g;
  gm.K = (int64_t)nk * BK;
  int ksplit, kb_per;
  choose_split(gm, &ksplit, &kb_per, BN);
  if (const char* e = getenv("PFB_TC_KSPLIT")) ksplit_want = atoi(e);  // bring-up override
  if (ksplit_want > 0) {  // autotuner candidate / override: this many k-splits
    const int want = std::max(1, std::min(ksplit_want, kMaxCluster));
    kb_per = (nk + want - 1) / want;
    ksplit = (nk + kb_per - 1) / kb_per;
  }
  // TMA-store epilogue: C row-major with 16-byte aligned rows, overwrite
  CUtensorMap mc = f1.ah;
  int tma_store = 0;
  if (ksplit == 1 && !g.accumulate && g.scn == 1 && (g.N == 1 || (g.scm * 4) % 16 == 0) &&
      (g.batch == 1 || (g.scb * 4) % 16 == 0) &&
      (reinterpret_cast<uintptr_t>(g.C) & 15) == 0 && !getenv_flag("PFB_NO_TMA_STORE")) {
    const int64_t ldc = g.M == 1 ? (g.N + 3) / 4 * 4 : g.scm;
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)g.batch};
    cuuint64_t strides[2] = {(cuuint64_t)(ldc * 4),
                             (cuuint64_t)((g.batch == 1 ? ldc * g.M : g.scb) * 4)};
    cuuint32_t box[3] = {32, 32, 1};
    tma_store = encode(&mc, g.C, dims, strides, box) ? 1 : 0;
  }
  auto idesc_of = [](const PairFeed& f) {
    return C::IDESC | ((uint32_t)(f.am == kRawMN) << 15) | ((uint32_t)(f.bm == kRawMN) << 16);
  };
  const PairFeed& q = f2 ? *f2 : f1;
  Params p{(int)g.M, (int)g.N, nk * BK, (int)g.batch,
           (int)((g.M + BM - 1) / BM), (int)((g.N + BN - 1) / BN), f1.a_bc, f1.b_bc, f1.am, f1.bm,
           idesc_of(f1), g.C, g.scb, g.scm, g.scn, g.alpha_rows, g.accumulate, ksplit, kb_per,
           g.bias, g.sxb, g.sxm, g.sxn, g.act, 4096u, 512u, tma_store, tc_trace_buffer(),
           nk1, q.am, q.bm, q.a_bc, q.b_bc, idesc_of(q), g.dy, g.sdb, g.sdm, g.sdn, g.dop,
           chunk_kb(), getenv("PFB_TC_PRODUCTS") ? atoi(getenv("PFB_TC_PRODUCTS")) : 3,
           getenv("PFB_TC_EXP") ? atoi(getenv("PFB_TC_EXP")) : 0};
  const int64_t units = (int64_t)p.ntm * p.ntn * g.batch * ksplit;
  if (ksplit > 1) {
    // one CTA per (tile, k-split); the k-splits of a tile are one cluster
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)units);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)ksplit;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    kernel_launches()++;
    cudaLaunchKernelEx(&cfg, gemm_kernel<BN>, f1.ah, f1.al, f1.bh, f1.bl, mc, q.ah, q.al, q.bh, q.bl,
                       p);
  } else {
    const int grid = (int)std::min<int64_t>(units, num_sms());
    launch(gemm_kernel<BN>, grid, NUM_THREADS, C::SMEM_BYTES, s, f1.ah, f1.al, f1.bh, f1.bl, mc, q.ah,
           q.al, q.bh, q.bl, p);
  }
  return launch_status();
}

static int launch_bn(int bn, const GemmArgs& g, const PairFeed& f1, const PairFeed* f2,
                     cudaStream_t s, int ksplit_want) {
  if (bn == 32) return launch_gemm<32>(g, f1, f2, s, ksplit_want);
  if (bn == 64) return launch_gemm<64>(g, f1, f2, s, ksplit_want);
  return launch_gemm<128>(g, f1, f2, s, ksplit_want);
}

}  // namespace tc

int gemm_tcgen05(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s, int variant,
                 int ksplit_want, int bn) {
  using namespace tc;
  if (!gemm_tcgen05_eligible(g)) return PFB_E_UNSUPPORTED;
  if (variant == 0) variant = (2.0 * g.M * g.N * g.K * g.batch < 4e9) ? 2 : 1;
  if (const char* e = getenv("PFB_TC_VARIANT")) variant = atoi(e);  // experiments
  int am, bm;
  const int64_t need = pair_need(g, variant, &am, &bm);
  if (need > 0 && (ws == nullptr || ws_bytes < need)) return PFB_E_UNSUPPORTED;
  char* w = static_cast<char*>(ws);
  if (const char* e = getenv("PFB_TC_BN")) bn = atoi(e);  // experiments
  if (bn != 32 && bn != 64) bn = 128;
  PairFeed f;
  if (int e = prep_pair(g, variant, w, s, &f, bn)) return e;
  return launch_bn(bn, g, f, nullptr, s, ksplit_want);
}

int64_t gemm_tcgen05_dual_workspace(const GemmArgs& g1, const GemmArgs& g2) {
  return gemm_tcgen05_workspace(g1) + gemm_tcgen05_workspace(g2);
}

// C = epi(A1 B1 + A2 B2): both pairs accumulate into one TMEM tile (the
// K ranges are consecutive k-blocks of one launch); g1 carries C/epilogue.
int gemm_tcgen05_dual(const GemmArgs& g1, const GemmArgs& g2, void* ws, int64_t ws_bytes,
                      cudaStream_t s, int variant, int ksplit_want, int bn) {
  using namespace tc;
  if (!gemm_tcgen05_eligible(g1) || !gemm_tcgen05_eligible(g2)) return PFB_E_UNSUPPORTED;
  if (g1.M != g2.M || g1.N != g2.N || g1.batch != g2.batch || g2.kscale) return PFB_E_UNSUPPORTED;
  if (variant == 0) variant = (2.0 * g1.M * g1.N * (g1.K + g2.K) * g1.batch < 4e9) ? 2 : 1;
  int a1, b1, a2, b2;
  const int64_t need = pair_need(g1, variant, &a1, &b1) + pair_need(g2, variant, &a2, &b2);
  if (need > 0 && (ws == nullptr || ws_bytes < need)) return PFB_E_UNSUPPORTED;
  char* w = static_cast<char*>(ws);
  if (bn != 32 && bn != 64) bn = 128;
  PairFeed f1, f2;
  if (int e = prep_pair(g1, variant, w, s, &f1, bn)) return e;
  if (int e = prep_pair(g2, variant, w, s, &f2, bn)) return e;
  return launch_bn(bn, g1, f1, &f2, s, ksplit_want);
}

}  // namespace pfb

extern "C" int pfb_debug_tc_trace(unsigned long long* out16) {
  if (pfb::g_trace == nullptr) return PFB_E_UNSUPPORTED;
  cudaDeviceSynchronize();
  return cudaMemcpy(out16, pfb::g_trace, 512 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
                 cudaSuccess ? 0 : PFB_E_ARG;
}
