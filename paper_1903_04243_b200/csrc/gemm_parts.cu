// Split-K partials GEMM for skinny-M problems (pass F15, pfb_matmul_parts):
//
//   parts[s] = A[:, Ks] @ B[Ks, :]  (+ bias in s = 0)     s = 0..S-1
//
// One CTA per (128-row tile, BN-column tile, k-split).  Each split's K range
// (<= 8 k-blocks of 32) accumulates in 64-deep TMEM chunks summed in fp32
// registers (double-buffered TMEM: chunk c drains while c+1 multiplies); no
// reduction across splits: the consumer (a fused elementwise group) sums the
// S partials as it loads them.  This is the shape of the LSTM's per-step
// GEMMs (M = 256 examples, 128 of them per step, reference bench cell /
// BASELINE cfg4), where the reduced GEMM spent ~30% of its time in the
// cluster reduction (barriers waiting on the slowest CTA of the cluster, then
// DSMEM round trips).  BN = 128 by default: BN = 256 (every tcgen05.mma a
// 128x256x8 instruction, full TF32 issue rate -- 128-wide MMAs cost ~60
// cycles each regardless of N, tools/experiments/mma_rate.cu) doubles the
// partials the consumer must read and measured slower on the cfg4 step
// (3.24 vs 2.69 ms, tools/experiments/parts_knobs.sh; PFB_PARTS_BN).
//
// 3xTF32 as in gemm_tcgen05.cu: A raw (the tensor core truncates it: hi =
// trunc(x); lo = rn(x - hi) written beside it in smem by the split warps),
// B as pre-split RN hi/lo planes; products A_hi B_hi + A_hi B_lo + A_lo B_hi.
// (Whole-split accumulation in TMEM -- 256 of K -- measured 2.9e-5 abs error
// on cfg4's gradients, outside atol 1e-5: the in-TMEM accumulation truncates;
// the 64-deep chunks bring it back to SIMT-fp32 level, tests/test_gpu_parts.py,
// tests/test_gpu_bench_scale.py.)
//
// Warps: 0 TMA producer, 1 TMEM allocator + MMA issuer, 2..9 split A tiles,
// then drain TMEM (warp w: lanes 32*(w%4).., columns half (w-2)/4) through a
// swizzled smem block and TMA-store 32x32 blocks of parts[s].
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "fused.cuh"
#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace pfb {
namespace tcs {

using namespace tc;

constexpr int BM = 128, BK = 32, UMMA_K = 8;
constexpr int A_BYTES = BM * BK * 4;  // 16 KB raw A tile (lo beside it)
constexpr int WARPS = 10, NUM_THREADS = 32 * WARPS, SPLIT_WARPS = 8;
constexpr int kMaxKb = 8;             // k-blocks per split
constexpr int CHUNK = 2;              // k-blocks per TMEM chunk (64 deep, then fp32 registers)

template <int BN>
struct Cfg {
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = BN == 256 ? 2 : 3;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static_assert(2 * BN <= 512, "double-buffered TMEM chunks");
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  static_assert(SMEM <= 232448, "shared memory");
  static_assert(SPLIT_WARPS * 4096 * (BN / 64) <= STAGES * STAGE, "epilogue staging reuses the stages");
};

struct Params {
  int M, N, nk, kb_per, ntn, S;
  int nk1;            // k-blocks of the first operand pair (dual GEMM: the rest from map_*2)
  const float* bias;  // split 0 only; broadcast strides
  int64_t sxm, sxn;
  unsigned long long* trace;  // PFB_TC_TRACE: phase stamps of CTA 0 + per-CTA start/end
};

__device__ __forceinline__ void pstamp(const Params& p, int i, bool cta_any = false) {
  if (p.trace != nullptr && (cta_any || blockIdx.x == 0)) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[i] = t;
  }
}

template <int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
parts_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_bh,
             const __grid_constant__ CUtensorMap map_bl, const __grid_constant__ CUtensorMap map_c,
             const __grid_constant__ CUtensorMap map_a2, const __grid_constant__ CUtensorMap map_bh2,
             const __grid_constant__ CUtensorMap map_bl2, Params p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* full = bars;                  // TMA -> split warps
  uint64_t* ready = bars + C::STAGES;     // split -> MMA
  uint64_t* empty = bars + 2 * C::STAGES; // MMA -> TMA
  uint64_t* acc_full = bars + 3 * C::STAGES;  // [2] MMA -> drain warps (chunk done)
  uint64_t* acc_empty = acc_full + 2;         // [2] drain warps -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x;
  const int s_idx = u % p.S, t = u / p.S;
  const int m0 = (t / p.ntn) * BM, n0 = (t % p.ntn) * BN;
  const int kb0 = s_idx * p.kb_per, kb1 = min(p.nk, kb0 + p.kb_per);
  const int nkb = kb1 - kb0;
  const int nch = (nkb + CHUNK - 1) / CHUNK;  // TMEM chunks (64 deep) of this split
  auto stage = [&](int s) { return smem + s * C::STAGE; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], SPLIT_WARPS);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], SPLIT_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bl)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) pstamp(p, 0);
  pdl_enter();
  if (threadIdx.x == 0) {
    pstamp(p, 1);
    if (blockIdx.x < 160) pstamp(p, 192 + blockIdx.x, true);
  }

  if (warp == 0) {
    if (lane == 0) {
      for (int g = 0; g < nkb; ++g) {
        const int s = g % C::STAGES, kb = kb0 + g;
        if (g >= C::STAGES) mbar_wait(&empty[s], ((g / C::STAGES) - 1) & 1);
        mbar_expect_tx(&full[s], A_BYTES + 2 * C::B_BYTES);
        const bool second = kb >= p.nk1;
        const int kc = (second ? kb - p.nk1 : kb) * BK;
        tma_load_3d(second ? &map_a2 : &map_a, &full[s], stage(s), kc, m0, 0);
        tma_load_3d(second ? &map_bh2 : &map_bh, &full[s], stage(s) + 2 * A_BYTES, kc, n0, 0);
        tma_load_3d(second ? &map_bl2 : &map_bl, &full[s], stage(s) + 2 * A_BYTES + C::B_BYTES, kc,
                    n0, 0);
        if (g < 8) pstamp(p, 16 + g);
      }
    }
  } else if (warp == 1) {
    // chunk c accumulates k-blocks [c*CHUNK, ..) into TMEM buffer c&1 (the
    // tensor core's in-TMEM accumulation truncates: 64-deep chunks summed in
    // fp32 registers keep the result at SIMT-fp32 accuracy, gemm_tcgen05.cu)
    int g = 0;
    for (int c = 0; c < nch; ++c) {
      const int buf = c & 1;
      if (c >= 2) mbar_wait(&acc_empty[buf], ((c >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t td = tmem + (uint32_t)(buf * BN);
      const int gend = min(nkb, (c + 1) * CHUNK);
      for (; g < gend; ++g) {
        const int s = g % C::STAGES;
        mbar_wait(&ready[s], (g / C::STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t ah = smem_desc_sw128(smem_u32(stage(s)));
        const uint64_t al = smem_desc_sw128(smem_u32(stage(s) + A_BYTES));
        const uint64_t bh = smem_desc_sw128(smem_u32(stage(s) + 2 * A_BYTES));
        const uint64_t bl = smem_desc_sw128(smem_u32(stage(s) + 2 * A_BYTES + C::B_BYTES));
        if (elect_one()) {
          if (g < 8) pstamp(p, 32 + g);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            const uint64_t d = (UMMA_K * 4) >> 4;  // +32 B inside the swizzle row
            const uint32_t acc = (g > c * CHUNK || k > 0) ? 1u : 0u;
            mma_tf32(td, ah + d * k, bh + d * k, C::IDESC, acc);
            mma_tf32(td, ah + d * k, bl + d * k, C::IDESC, 1u);
            mma_tf32(td, al + d * k, bh + d * k, C::IDESC, 1u);
          }
          mma_commit(&empty[s]);
          if (g == gend - 1) mma_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else {
    const int et = threadIdx.x - 64;  // 0..255
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row0 = m0 + quarter * 32;
    constexpr int DC = BN / 2;  // accumulator columns per warp
    float acc[DC];
    // split 0 starts from the bias (row-broadcast or full matrix)
    const bool add_bias = p.bias != nullptr && s_idx == 0;
#pragma unroll
    for (int j = 0; j < DC; ++j) {
      const int col = n0 + half * DC + j;
      acc[j] = (add_bias && row0 + lane < p.M && col < p.N)
                   ? __ldg(p.bias + (int64_t)(row0 + lane) * p.sxm + (int64_t)col * p.sxn)
                   : 0.f;
    }
    int g = 0;
    auto drain = [&](int c) {
      const int buf = c & 1;
      mbar_wait(&acc_full[buf], (c >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int cc = 0; cc < DC; cc += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * BN + half * DC + cc), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[cc + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    };
    // split chunk c's stages, then drain chunk c-1 (the MMA works on chunk
    // c-1 while chunk c is split)
    for (int c = 0; c < nch; ++c) {
      const int gend = min(nkb, (c + 1) * CHUNK);
      for (; g < gend; ++g) {
        const int s = g % C::STAGES;
        mbar_wait(&full[s], (g / C::STAGES) & 1);
        if (et == 0 && g < 8) pstamp(p, 48 + g);
        split_tf32_smem(smem_u32(stage(s)), smem_u32(stage(s) + A_BYTES), A_BYTES / 16, et,
                        32 * SPLIT_WARPS);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&ready[s]);
      }
      if (c > 0) drain(c - 1);
    }
    drain(nch - 1);
    if (et == 0) pstamp(p, 2);
    // ---- epilogue: registers -> swizzled 32x32 blocks (one per 32 columns;
    // the stage memory is idle now) -> TMA store of parts[s_idx]
    constexpr int NB = DC / 32;
    float* blk0 = reinterpret_cast<float*>(smem) + (warp - 2) * 1024 * NB;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int col0 = n0 + half * DC + 32 * b;
      float* blk = blk0 + 1024 * b;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(blk + lane * 32 + 4 * (q ^ (lane & 7))) =
            make_float4(acc[32 * b + 4 * q], acc[32 * b + 4 * q + 1], acc[32 * b + 4 * q + 2],
                        acc[32 * b + 4 * q + 3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&map_c, blk, col0, row0, s_idx);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (et == 0) pstamp(p, 3);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) {
    pstamp(p, 4);
    if (blockIdx.x < 160) pstamp(p, 352 + blockIdx.x, true);
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}

// K-split count: enough (tile, split) units to cover the SMs, <= kMaxKb
// k-blocks (TMEM accumulation depth) per split, >= 2 k-blocks each
static int plan(int64_t M, int64_t N, int64_t K, int BN, int* kb_per) {
  static const int smax = [] {  // PFB_PARTS_SMAX: cap on S (experiments)
    const char* e = getenv("PFB_PARTS_SMAX");
    return e ? std::max(1, atoi(e)) : kMaxParts;
  }();
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int64_t nk = ((K + 3) / 4 * 4 + BK - 1) / BK;
  int64_t S = std::min<int64_t>(smax, std::max<int64_t>(1, 148 / tiles));
  S = std::max<int64_t>(S, (nk + kMaxKb - 1) / kMaxKb);  // TMEM depth bound
  S = std::min<int64_t>(S, std::max<int64_t>(1, nk / 2));
  int64_t per = (nk + S - 1) / S;
  S = (nk + per - 1) / per;
  if (per > kMaxKb || S * tiles > 4 * 148) return 0;
  *kb_per = (int)per;
  return (int)S;
}

template <int BN>
static int launch(const GemmArgs& g, const CUtensorMap* maps, int nk1, int nk, int S, int kb_per,
                  cudaStream_t s) {
  using C = Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(parts_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  Params p;
  p.M = (int)g.M; p.N = (int)g.N;
  p.nk = nk;
  p.nk1 = nk1;
  p.kb_per = kb_per;
  p.ntn = (int)((g.N + BN - 1) / BN);
  p.S = S;
  p.bias = g.bias; p.sxm = g.sxm; p.sxn = g.sxn;
  p.trace = tc_trace_buffer();
  const int units = (int)(((g.M + BM - 1) / BM) * p.ntn * S);
  pfb::launch(parts_kernel<BN>, dim3(units), dim3(NUM_THREADS), C::SMEM, s, maps[0], maps[1],
              maps[2], maps[3], maps[4], maps[5], maps[6], p);
  return launch_status();
}

static int64_t kblocks(const GemmArgs& g) { return ((g.K + 3) / 4 * 4 + BK - 1) / BK; }

// A K-major and TMA-readable as is, batch 1, no prologue / epilogue beyond a bias
static bool parts_operand_ok(const GemmArgs& g) {
  if (g.batch != 1 || g.M < 1 || g.N < 8 || g.K < 8 || g.kscale || g.accumulate || g.act ||
      g.dop || g.alpha_rows)
    return false;
  return g.sak == 1 && (g.M == 1 || ((g.sam * 4) % 16 == 0 && g.sam >= g.K)) &&
         (reinterpret_cast<uintptr_t>(g.A) & 15) == 0;
}

}  // namespace tcs

static int parts_bn(const GemmArgs& g) {
  static const int env = [] {
    const char* e = getenv("PFB_PARTS_BN");
    return e ? atoi(e) : 0;
  }();
  if (env == 128 || env == 256) return env;
  return 128;
}

// S for pfb_matmul_parts (0: not applicable); g2 (nullable): the second
// operand pair of a dual GEMM (K ranges concatenated, same M, N)
int gemm_parts_count(const GemmArgs& g, const GemmArgs* g2) {
  using namespace tcs;
  if (!parts_operand_ok(g) || (g2 && (!parts_operand_ok(*g2) || g2->M != g.M || g2->N != g.N)))
    return 0;
  const int64_t nk = kblocks(g) + (g2 ? kblocks(*g2) : 0);
  // small products (cfg1's 32x256x784 forward) stay on the autotuned paths:
  // the partials cost their consumers S reads and win only where the k-loop
  // and the cluster reduction are long (cfg4's per-step GEMMs: >= 268M MACs)
  if (nk < 2 || (double)g.M * g.N * nk * BK < (double)(1 << 26)) return 0;
  if (g.N % 4 != 0) return 0;  // the [S, M, N] partials' rows must be 16-byte aligned (TMA store)
  int per;
  return plan(g.M, g.N, nk * BK, parts_bn(g), &per);
}

int64_t gemm_parts_workspace(const GemmArgs& g, const GemmArgs* g2) {
  auto one = [](const GemmArgs& x) -> int64_t {
    if (x.b_hi) return 0;
    const int64_t Kp = (x.K + 3) / 4 * 4;
    return 2 * ((x.N * Kp * 4 + 255) / 256 * 256);
  };
  return one(g) + (g2 ? one(*g2) : 0);
}

// the A map and the B hi / lo maps of one operand pair (B split into the
// workspace at `w` when it has no pre-split planes)
static int pair_maps(const GemmArgs& g, int BN, char*& w, cudaStream_t s, CUtensorMap* m) {
  using namespace tcs;
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const float* bh = g.b_hi;
  const float* bl = g.b_lo;
  if (!bh) {
    float* h = reinterpret_cast<float*>(w);
    w += (g.N * Kp * 4 + 255) / 256 * 256;
    float* l = reinterpret_cast<float*>(w);
    w += (g.N * Kp * 4 + 255) / 256 * 256;
    tc_split_launch(g.B, 1, g.N, g.K, Kp, 0, g.sbn, g.sbk, h, l, nullptr, 0, 0, s);
    bh = h;
    bl = l;
  }
  {
    const int64_t ld = g.M == 1 ? Kp : g.sam;
    cuuint64_t dims[3] = {(cuuint64_t)g.K, (cuuint64_t)g.M, 1};
    cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)(ld * g.M * 4)};
    cuuint32_t box[3] = {BK, BM, 1};
    if (!encode(&m[0], g.A, dims, strides, box)) return PFB_E_UNSUPPORTED;
  }
  cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)g.N, 1};
  cuuint64_t strides[2] = {(cuuint64_t)(Kp * 4), (cuuint64_t)(g.N * Kp * 4)};
  cuuint32_t box[3] = {BK, (cuuint32_t)BN, 1};
  if (!encode(&m[1], bh, dims, strides, box) || !encode(&m[2], bl, dims, strides, box))
    return PFB_E_UNSUPPORTED;
  return 0;
}

int gemm_parts(const GemmArgs& g, const GemmArgs* g2, int S, float* parts, int64_t part_stride,
               int64_t ldc, void* ws, int64_t ws_bytes, cudaStream_t s) {
  using namespace tcs;
  const int BN = parts_bn(g);
  const int nk1 = (int)kblocks(g), nk = nk1 + (g2 ? (int)kblocks(*g2) : 0);
  int kb_per = 0;
  if (gemm_parts_count(g, g2) != S || plan(g.M, g.N, (int64_t)nk * BK, BN, &kb_per) != S)
    return PFB_E_UNSUPPORTED;
  if ((part_stride * 4) % 16 != 0 || (ldc * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(parts) & 15))
    return PFB_E_UNSUPPORTED;
  const int64_t need = gemm_parts_workspace(g, g2);
  if (need > 0 && (ws == nullptr || ws_bytes < need)) return PFB_E_UNSUPPORTED;
  char* w = static_cast<char*>(ws);
  CUtensorMap maps[7];  // A, B hi, B lo, C, A2, B2 hi, B2 lo
  if (int e = pair_maps(g, BN, w, s, &maps[0])) return e;
  if (g2) {
    if (int e = pair_maps(*g2, BN, w, s, &maps[4])) return e;
  } else {
    maps[4] = maps[0]; maps[5] = maps[1]; maps[6] = maps[2];  // unused (nk1 == nk)
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)S};
    cuuint64_t strides[2] = {(cuuint64_t)(ldc * 4), (cuuint64_t)(part_stride * 4)};
    cuuint32_t box[3] = {32, 32, 1};
    if (!encode(&maps[3], parts, dims, strides, box)) return PFB_E_UNSUPPORTED;
  }
  return BN == 256 ? tcs::launch<256>(g, maps, nk1, nk, S, kb_per, s)
                   : tcs::launch<128>(g, maps, nk1, nk, S, kb_per, s);
}

}  // namespace pfb
