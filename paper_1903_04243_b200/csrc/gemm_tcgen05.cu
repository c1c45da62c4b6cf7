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

namespace pfb {
namespace tc {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, UMMA_K = 8;
constexpr int CHUNK_KB = 2;                       // k-blocks accumulated in TMEM per chunk
constexpr int TILE_BYTES = BM * BK * 4;           // 16 KB per operand tile
constexpr int STAGE_BYTES = 4 * TILE_BYTES;       // A_hi, A_lo, B_hi, B_lo
constexpr int EPI_WARPS = 8;                      // 2 per TMEM lane quarter, 64 columns each
constexpr int EPI_COLS = BN / 2;
constexpr int EPI_STAGE_FLOATS = 32 * 32;         // per epilogue warp: one 32x32 block,
                                                  // 16B chunks XOR-swizzled by row
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                           EPI_WARPS * EPI_STAGE_FLOATS * 4;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;  // TMA, MMA, 8 epilogue warps
constexpr int TMEM_COLS = 2 * BN;                 // double-buffered chunk accumulator

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// K-major, 128B-swizzled operand tile: 8-row atoms of 1024 B (SBO), version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);          // start address
  d |= (uint64_t)(16 >> 4) << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // SBO: stride between 8-row atoms
  d |= (uint64_t)1 << 46;                          // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
  return d;
}

// kind::tf32, D=f32, K-major A and B, M=128, N=BN
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

// ---------------------------------------------------------------------------
// split: x (view [batch, rows, K], any strides) -> dense hi, lo [batch, rows, Kp]

__global__ void __launch_bounds__(256) split_kernel(const float* __restrict__ x, int64_t rows,
                                                    int64_t K, int64_t Kp, int64_t sb, int64_t sr,
                                                    int64_t sk, float* __restrict__ hi,
                                                    float* __restrict__ lo) {
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
      lb[r * Kp + k] = to_tf32(v - h);
    }
  }
}

struct Params {
  int M, N, K, batch;
  int ntm, ntn;
  int a_bcast, b_bcast;  // operand shared across the batch (split once)
  float* C;
  int64_t scb, scm, scn;
  const float* alpha_rows;
  int accumulate;
  int ksplit;            // >1: work unit = (tile, k-range); partial tiles -> `partials`
  int kb_per_split;      // k-blocks per split (multiple of CHUNK_KB)
  float* partials;       // [ksplit][batch][M][N] when ksplit > 1
};

__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_ah, const __grid_constant__ CUtensorMap map_al,
            const __grid_constant__ CUtensorMap map_bh, const __grid_constant__ CUtensorMap map_bl,
            Params p) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = bars;                   // [STAGES] TMA -> MMA
  uint64_t* empty = bars + STAGES;         // [STAGES] MMA -> TMA
  uint64_t* acc_full = bars + 2 * STAGES;  // [2] MMA -> accumulators
  uint64_t* acc_empty = acc_full + 2;      // [2] accumulators -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (p.K + BK - 1) / BK;
  const int tiles_per_batch = p.ntm * p.ntn;
  const int ntiles = tiles_per_batch * p.batch * p.ksplit;  // work units

  auto tile = [&](int s, int which) { return smem + s * STAGE_BYTES + which * TILE_BYTES; };
  // which: 0 = A_hi, 1 = A_lo, 2 = B_hi, 3 = B_lo

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 32 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ah)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_al)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bh)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bl)) : "memory");
      int g = 0;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
        const int t = u / p.ksplit, ks = u % p.ksplit;
        const int bz = t / tiles_per_batch, r = t % tiles_per_batch;
        const int m0 = (r / p.ntn) * BM, n0 = (r % p.ntn) * BN;
        const int za = p.a_bcast ? 0 : bz, zb = p.b_bcast ? 0 : bz;
        const int kb0 = ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
          mbar_expect_tx(&full[s], 4 * TILE_BYTES);
          tma_load_3d(&map_ah, &full[s], tile(s, 0), kb * BK, m0, za);
          tma_load_3d(&map_al, &full[s], tile(s, 1), kb * BK, m0, za);
          tma_load_3d(&map_bh, &full[s], tile(s, 2), kb * BK, n0, zb);
          tma_load_3d(&map_bl, &full[s], tile(s, 3), kb * BK, n0, zb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int g = 0, gc = 0;
      for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
        const int ks = u % p.ksplit;
        const int kb0 = ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
        const int uchunks = (kb1 - kb0 + CHUNK_KB - 1) / CHUNK_KB;
        for (int c = 0; c < uchunks; ++c, ++gc) {
          const int buf = gc & 1;
          if (gc >= 2) mbar_wait(&acc_empty[buf], ((gc >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t tmem_d = tmem_base + (uint32_t)(buf * BN);
          const int kb_beg = kb0 + c * CHUNK_KB;
          const int kb_end = min(kb1, kb_beg + CHUNK_KB);
          for (int kb = kb_beg; kb < kb_end; ++kb, ++g) {
            const int s = g % STAGES;
            mbar_wait(&full[s], (g / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t a_hi = smem_desc_sw128(smem_u32(tile(s, 0)));
            const uint64_t a_lo = smem_desc_sw128(smem_u32(tile(s, 1)));
            const uint64_t b_hi = smem_desc_sw128(smem_u32(tile(s, 2)));
            const uint64_t b_lo = smem_desc_sw128(smem_u32(tile(s, 3)));
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t adv = (uint64_t)((k * UMMA_K * 4) >> 4);  // +32 B along K
              const uint32_t acc = (kb > kb_beg || k > 0) ? 1u : 0u;
              mma_tf32(tmem_d, a_hi + adv, b_hi + adv, acc);
              mma_tf32(tmem_d, a_hi + adv, b_lo + adv, 1u);
              mma_tf32(tmem_d, a_lo + adv, b_hi + adv, 1u);
            }
            mma_commit(&empty[s]);
          }
          mma_commit(&acc_full[buf]);
        }
      }
    }
    __syncwarp();
  } else {
    // ---- accumulators + epilogue (warps 2..9): warp w owns TMEM lanes
    // 32*(w%4)..+31 (its rows) and columns [half*64, half*64+64) ----
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    float* stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256) +
                   (warp - 2) * EPI_STAGE_FLOATS;
    int gc = 0;
    for (int u = blockIdx.x; u < ntiles; u += gridDim.x) {
      const int t = u / p.ksplit, ks = u % p.ksplit;
      const int bz = t / tiles_per_batch, r = t % tiles_per_batch;
      const int m0 = (r / p.ntn) * BM, n0 = (r % p.ntn) * BN;
      const int kb0 = ks * p.kb_per_split, kb1 = min(nk, kb0 + p.kb_per_split);
      const int uchunks = (kb1 - kb0 + CHUNK_KB - 1) / CHUNK_KB;
      float acc[EPI_COLS];
#pragma unroll
      for (int j = 0; j < EPI_COLS; ++j) acc[j] = 0.f;
      for (int c = 0; c < uchunks; ++c, ++gc) {
        const int buf = gc & 1;
        mbar_wait(&acc_full[buf], (gc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int cc = 0; cc < EPI_COLS; cc += 32) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) +
                        (uint32_t)(buf * BN + half * EPI_COLS + cc), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[cc + j] += __uint_as_float(v[j]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(&acc_empty[buf]);
      }
      // 32x32 blocks through smem: each lane writes its row as float4s, then
      // every store instruction covers 4 rows x 128 contiguous bytes
      const int row0 = m0 + quarter * 32;
      const bool partial = p.ksplit > 1;  // dense partial tile, epilogue in the reduction
      float* cbase = partial ? p.partials + ((int64_t)ks * p.batch + bz) * p.M * p.N
                             : p.C + bz * p.scb;
      const int64_t ldm = partial ? p.N : p.scm, ldn = partial ? 1 : p.scn;
      const int sub_r = lane >> 3, sub_c = (lane & 7) * 4;
#pragma unroll
      for (int cc = 0; cc < EPI_COLS; cc += 32) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stage + lane * 32 + 4 * (q ^ (lane & 7))) =
              make_float4(acc[cc + 4 * q], acc[cc + 4 * q + 1], acc[cc + 4 * q + 2],
                          acc[cc + 4 * q + 3]);
        __syncwarp();
        const int col = n0 + half * EPI_COLS + cc + sub_c;
#pragma unroll 4
        for (int i = 0; i < 32; i += 4) {
          const int row = row0 + i + sub_r;
          if (row < p.M) {
            const float alpha = (!partial && p.alpha_rows)
                                    ? __ldg(p.alpha_rows + (int64_t)bz * p.M + row) : 1.f;
            const int srow = i + sub_r;
            float4 v = *reinterpret_cast<const float4*>(
                stage + srow * 32 + 4 * ((sub_c >> 2) ^ (srow & 7)));
            v.x *= alpha; v.y *= alpha; v.z *= alpha; v.w *= alpha;
            float* q = cbase + (int64_t)row * ldm + (int64_t)col * ldn;
            if (ldn == 1 && col + 3 < p.N && ((reinterpret_cast<uintptr_t>(q) & 15) == 0)) {
              if (p.accumulate && !partial) {
                const float4 o = *reinterpret_cast<const float4*>(q);
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              *reinterpret_cast<float4*>(q) = v;
            } else {
              const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                if (col + j < p.N) {
                  float* qq = q + (int64_t)j * ldn;
                  *qq = (p.accumulate && !partial) ? *qq + e[j] : e[j];
                }
              }
            }
          }
        }
        __syncwarp();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// --- host side -------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// dense K-major plane [batch][rows][Kp]
static bool make_map(CUtensorMap* map, const float* base, int64_t Kp, int64_t rows, int64_t batch) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(Kp * 4), (cuuint64_t)(rows * Kp * 4)};
  cuuint32_t box[3] = {BK, BM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
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

// K-splits so that (tiles x splits) covers the SMs, >= 2 chunks per split
static void choose_split(const GemmArgs& g, int* ksplit, int* kb_per) {
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
    return waves * (per * 0.6 + 1.5) + (real > 1 ? 4.0 : 0.0);
  };
  int best_per = 0;
  double best = cost(1, &best_per);
  int s_max = 1;
  if (tiles < num_sms() && nk >= 4 * CHUNK_KB)
    s_max = (int)std::max<int64_t>(1, std::min<int64_t>(
        std::min<int64_t>((num_sms() + tiles - 1) / tiles, nk / (2 * CHUNK_KB)), 32));
  for (int s = 2; s <= s_max; ++s) {
    int per;
    const double c = cost(s, &per);
    if (c < best) { best = c; best_per = per; }
  }
  *kb_per = best_per;
  *ksplit = (nk + best_per - 1) / best_per;
}

__global__ void __launch_bounds__(256) splitk_sum(int64_t M, int64_t N, int64_t batch, int ksplit,
                                                  const float* __restrict__ part, float* C,
                                                  int64_t scb, int64_t scm, int64_t scn,
                                                  const float* alpha_rows, int accumulate) {
  pdl_enter();
  const int64_t plane = batch * M * N;
  const int64_t total = plane;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < ksplit; ++k) s += __ldg(part + k * plane + i);
    const int64_t b = i / (M * N), rem = i - b * M * N;
    const int64_t m = rem / N, n = rem - m * N;
    if (alpha_rows) s *= alpha_rows[b * M + m];
    float* q = C + b * scb + m * scm + n * scn;
    *q = accumulate ? *q + s : s;
  }
}

}  // namespace tc

// Workspace: hi/lo planes of both operands (K padded to a multiple of 4 so
// every TMA row stride is 16-byte aligned).
int64_t gemm_tcgen05_workspace(const GemmArgs& g) {
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int64_t ba = (g.sab == 0 && g.batch > 1) ? 1 : g.batch;
  const int64_t bb = (g.sbb == 0 && g.batch > 1) ? 1 : g.batch;
  int ks, per;
  tc::choose_split(g, &ks, &per);
  const int64_t part = ks > 1 ? tc::align_up((int64_t)ks * g.batch * g.M * g.N * 4) : 0;
  return 2 * tc::align_up(ba * g.M * Kp * 4) + 2 * tc::align_up(bb * g.N * Kp * 4) + part;
}

bool gemm_tcgen05_eligible(const GemmArgs& g) {
  if (g.K < 8 || g.M < 1 || g.N < 8) return false;
  return !(g.M > (1ll << 31) || g.N > (1ll << 31) || g.K > (1ll << 31) || g.batch > 65535 ||
           (g.M + 31) / 32 > 65535 || (g.N + 31) / 32 > 65535);
}

// Dispatch model (microseconds), calibrated on B200 (tools/gemm_probe.py):
// tensor path ~0.45 us per 32-deep k-block per 128x128 tile per wave plus
// fixed split/launch costs; SIMT fp32 ~15 TFLOP/s.  Skinny problems with few
// tiles (batch-128 forward passes) go SIMT with split-K.
bool gemm_tcgen05_profitable(const GemmArgs& g) {
  if (g.K < 16 || g.M < 16 || g.N < 16) return false;
  const double tiles = (double)((g.M + 127) / 128) * ((g.N + 127) / 128) * g.batch;
  int ks, per;
  tc::choose_split(g, &ks, &per);
  const double nk = (double)per;
  const double waves = std::ceil(tiles * ks / tc::num_sms());
  const double t_tc = waves * (nk * 0.6 + 1.5) + 6.0 + (ks > 1 ? 4.0 : 0.0);
  const double t_simt = 2.0 * g.M * g.N * g.K * g.batch / 15e6 + 3.0;
  return t_tc < t_simt;
}

int gemm_tcgen05(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s) {
  using namespace tc;
  if (!gemm_tcgen05_eligible(g)) return PFB_E_UNSUPPORTED;
  if (ws == nullptr || ws_bytes < gemm_tcgen05_workspace(g)) return PFB_E_UNSUPPORTED;
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int a_bc = g.sab == 0 && g.batch > 1, b_bc = g.sbb == 0 && g.batch > 1;
  const int64_t ba = a_bc ? 1 : g.batch, bb = b_bc ? 1 : g.batch;
  char* w = static_cast<char*>(ws);
  float* ah = reinterpret_cast<float*>(w); w += align_up(ba * g.M * Kp * 4);
  float* al = reinterpret_cast<float*>(w); w += align_up(ba * g.M * Kp * 4);
  float* bh = reinterpret_cast<float*>(w); w += align_up(bb * g.N * Kp * 4);
  float* bl = reinterpret_cast<float*>(w); w += align_up(bb * g.N * Kp * 4);
  int ksplit, kb_per;
  choose_split(g, &ksplit, &kb_per);
  float* partials = ksplit > 1 ? reinterpret_cast<float*>(w) : nullptr;
  // split (and re-layout) both operands; padded K columns are written as 0
  dim3 ga((unsigned)((Kp + 31) / 32), (unsigned)((g.M + 31) / 32), (unsigned)ba);
  dim3 gb((unsigned)((Kp + 31) / 32), (unsigned)((g.N + 31) / 32), (unsigned)bb);
  launch(split_kernel, ga, 256, 0, s, g.A, g.M, g.K, Kp, g.sab, g.sam, g.sak, ah, al);
  launch(split_kernel, gb, 256, 0, s, g.B, g.N, g.K, Kp, g.sbb, g.sbn, g.sbk, bh, bl);
  CUtensorMap mah, mal, mbh, mbl;
  if (!make_map(&mah, ah, Kp, g.M, ba) || !make_map(&mal, al, Kp, g.M, ba) ||
      !make_map(&mbh, bh, Kp, g.N, bb) || !make_map(&mbl, bl, Kp, g.N, bb))
    return PFB_E_UNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  Params p{(int)g.M, (int)g.N, (int)Kp, (int)g.batch,
           (int)((g.M + BM - 1) / BM), (int)((g.N + BN - 1) / BN), a_bc, b_bc,
           g.C, g.scb, g.scm, g.scn, g.alpha_rows, g.accumulate, ksplit, kb_per, partials};
  const int64_t units = (int64_t)p.ntm * p.ntn * g.batch * ksplit;
  const int grid = (int)std::min<int64_t>(units, num_sms());
  launch(gemm_kernel, grid, NUM_THREADS, SMEM_BYTES, s, mah, mal, mbh, mbl, p);
  if (ksplit > 1)
    launch(splitk_sum, grid_for(g.batch * g.M * g.N, 256), 256, 0, s, g.M, g.N, g.batch, ksplit,
           (const float*)partials, g.C, g.scb, g.scm, g.scn, g.alpha_rows, g.accumulate);
  return launch_status();
}

}  // namespace pfb
