// fp32-accurate GEMM on CTA pairs: tcgen05.mma.cta_group::2 kind::tf32 with
// the 3xTF32 split (see gemm_tcgen05.cu for the numerics), 256-row pair tiles.
//
// Why pairs: the 1-CTA kernel with 128x128 tiles needs 4 operand tiles
// (A_hi, A_lo, B_hi, B_lo) per 32-deep k-block for 12 UMMAs of 64 cycles;
// chip-wide that is ~2x what L2/TMA delivers, so it is feed-bound at ~30-65%
// of the 3xTF32 peak.  A CTA pair issues UMMA 256xBNx8 (BN = 128 or 256):
// each CTA loads its own 128 rows of A and BN/2 rows of B -- raw fp32, split
// into hi/lo in its own shared memory -- and the leader CTA's single MMA
// thread drives both SMs' tensor cores from both CTAs' tiles.  Per SM and
// k-block that is 16 KB + BN/2*128 B of L2 traffic for 12 UMMAs of BN/2
// cycles: 3-4x less operand traffic per flop than the 1-CTA kernel.
//
// Per CTA, 10 warps:
//   warp 0     TMA producer (own A rows, own half of B), STAGES-deep ring
//   warp 1     TMEM allocator (cta_group::2, both CTAs); leader: MMA issuer
//   warps 2-9  split raw tiles in smem (hi in place, lo beside it) and signal
//              the leader's `ready` barrier (remote mbarrier arrive); drain
//              finished TMEM chunks into fp32 registers (round-to-nearest sum
//              of 128-deep chunks, see the truncation note in gemm_tcgen05.cu)
//              and release them on the leader's `acc_empty`; TMA-store the
//              finished 128 x BN half tile of this CTA.
// Barriers: full/empty per stage are CTA-local (TMA tx / multicast commit);
// ready and acc_empty live in the leader (16 remote warp arrivals each);
// acc_full is signalled in both CTAs by the multicast commit.
#include <algorithm>
#include <cmath>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace pfb {
namespace tcp {

using namespace tc;

constexpr int BK = 32, UMMA_K = 8, EPI_WARPS = 8;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
// TMEM-resident mode: 4 more warps split the raw stages, so splitting the
// next tile never waits behind the drain + store of the previous one
constexpr int SPLIT_WARPS = 4;
template <bool SINGLE>
constexpr int threads_of() { return NUM_THREADS + (SINGLE ? 32 * SPLIT_WARPS : 0); }
constexpr int A_BYTES = 128 * BK * 4;  // 16 KB: this CTA's 128 rows of A
enum { kPreSplit = 0, kRawK = 1, kRawMN = 2 };

// TMEM-resident mode (SINGLE, short K): the epilogue is store-bound, so the
// 256-wide tile trades a stage for a second staging block per warp (a
// block's TMA store drains while the next one is written)
template <int BN, bool SINGLE = false>
struct Cfg {
  static constexpr int BNH = BN / 2;                 // B rows held by each CTA
  static constexpr int B_BYTES = BNH * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = BN == 256 ? (SINGLE ? 2 : 3) : 4;
  static constexpr int EPI_COLS = BN / 2;            // accumulator columns per epilogue warp
  static constexpr int NSTG = (BN == 256 && SINGLE) ? 2 : 1;  // staging blocks per warp
  static constexpr int STAGING = EPI_WARPS * 32 * 32 * 4 * NSTG;
  static constexpr int SMEM = STAGES * STAGE_BYTES + STAGING + 1024 + 256;
  static constexpr int TMEM_COLS = 2 * BN;           // double-buffered chunk accumulator
};

struct PParams {
  int M, N, K, batch;
  int ntm, ntn;  // pair tiles along M (256 rows) and N (BN columns)
  int a_bcast, b_bcast, a_mode, b_mode;
  uint32_t idesc;
  float* C;
  int64_t scb, scm, scn;
  const float* alpha_rows;
  int accumulate;
  const float* bias;
  int64_t sxb, sxm, sxn;
  int act;
  int tma_store;
  int chunk_kb;
  const float* dy;  // derivative epilogue (GemmArgs::dop)
  int64_t sdb, sdm, sdn;
  int dop;
  unsigned long long* trace;  // PFB_TC_TRACE stamps of CTA 0 (bring-up)
};

__device__ __forceinline__ void pstamp(const PParams& p, int i) {
  if (p.trace != nullptr && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[i] = t;
  }
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// arrive on the barrier at the same smem offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t da, uint64_t db,
                                              uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// completion of all prior MMAs arrives on `bar` in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void load_operand(const CUtensorMap* mh, const CUtensorMap* ml, int mode,
                                             uint64_t* bar, uint8_t* dst_hi, uint8_t* dst_lo,
                                             int kb, int row0, int z, int rows) {
  if (mode == kRawMN) {
    for (int j = 0; j < rows / 32; ++j)
      tma_load_3d(mh, bar, dst_hi + j * 4096, row0 + 32 * j, kb * BK, z);
  } else {
    tma_load_3d(mh, bar, dst_hi, kb * BK, row0, z);
    if (mode == kPreSplit) tma_load_3d(ml, bar, dst_lo, kb * BK, row0, z);
  }
}

__device__ __forceinline__ void epi4(const PParams& p, int bz, int row, int col, float4& v) {
  if (p.bias == nullptr && p.act == 0 && p.dop == 0) return;
  float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (p.bias && col + j < p.N)
      e[j] += __ldg(p.bias + (int64_t)bz * p.sxb + (int64_t)row * p.sxm + (int64_t)(col + j) * p.sxn);
    e[j] = apply_act(p.act, e[j]);
    if (p.dop && col + j < p.N)
      e[j] *= dop_factor(p.dop, p.dy,
                         (int64_t)bz * p.sdb + (int64_t)row * p.sdm + (int64_t)(col + j) * p.sdn);
  }
  v = make_float4(e[0], e[1], e[2], e[3]);
}

template <int BN, bool SINGLE>
__global__ void __launch_bounds__(threads_of<SINGLE>(), 1)
pair_kernel(const __grid_constant__ CUtensorMap map_ah, const __grid_constant__ CUtensorMap map_al,
            const __grid_constant__ CUtensorMap map_bh, const __grid_constant__ CUtensorMap map_bl,
            const __grid_constant__ CUtensorMap map_c, PParams p) {
  using C = Cfg<BN, SINGLE>;
  constexpr int STAGES = C::STAGES, BNH = C::BNH, EPI_COLS = C::EPI_COLS;
  if (threadIdx.x == 0) pstamp(p, 0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* staging = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES + C::STAGING);
  uint64_t* full = bars;                   // [STAGES] local TMA -> local split warps
  uint64_t* empty = bars + STAGES;         // [STAGES] MMA (multicast commit) -> local TMA
  uint64_t* ready = bars + 2 * STAGES;     // [STAGES] leader: both CTAs' split warps -> MMA
  uint64_t* acc_full = bars + 3 * STAGES;  // [2] MMA (multicast) -> both CTAs' epilogues
  uint64_t* acc_empty = acc_full + 2;      // [2] leader: both CTAs' epilogues -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = (int)(blockIdx.x >> 1), npairs = (int)(gridDim.x >> 1);
  const int nk = (p.K + BK - 1) / BK;
  const int tiles_per_batch = p.ntm * p.ntn;
  const int units = tiles_per_batch * p.batch;
  const int chunk = SINGLE ? nk : p.chunk_kb;

  auto tile = [&](int s, int which) -> uint8_t* {  // 0 A_hi, 1 A_lo, 2 B_hi, 3 B_lo
    uint8_t* b = smem + s * C::STAGE_BYTES;
    return which < 2 ? b + which * A_BYTES : b + 2 * A_BYTES + (which - 2) * C::B_BYTES;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], 2);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ah)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bh)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // peers' barriers are initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();  // prologue above overlaps the previous kernel (PDL)
  if (threadIdx.x == 0) pstamp(p, 1);

  const int bytes_a = (p.a_mode == kPreSplit ? 2 : 1) * A_BYTES;
  const int bytes_b = (p.b_mode == kPreSplit ? 2 : 1) * C::B_BYTES;

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int u = pair; u < units; u += npairs) {
        const int bz = u / tiles_per_batch, r = u % tiles_per_batch;
        const int m0 = (r / p.ntn) * 256 + (int)rank * 128;
        const int n0 = (r % p.ntn) * BN + (int)rank * BNH;
        const int za = p.a_bcast ? 0 : bz, zb = p.b_bcast ? 0 : bz;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % STAGES;
          if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
          mbar_expect_tx(&full[s], bytes_a + bytes_b);
          load_operand(&map_ah, &map_al, p.a_mode, &full[s], tile(s, 0), tile(s, 1), kb, m0, za, 128);
          load_operand(&map_bh, &map_bl, p.b_mode, &full[s], tile(s, 2), tile(s, 3), kb, n0, zb, BNH);
          if (g == 0) pstamp(p, 2);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      const bool amn = p.a_mode == kRawMN, bmn = p.b_mode == kRawMN;
      // k-step advance: +32 B inside the swizzle row (K-major) or one 1 KB atom (MN-major)
      const uint64_t astep = amn ? (1024 >> 4) : ((UMMA_K * 4) >> 4);
      const uint64_t bstep = bmn ? (1024 >> 4) : ((UMMA_K * 4) >> 4);
      const bool lo_lo = p.a_mode != kPreSplit && p.b_mode != kPreSplit;
      int g = 0, gc = 0;
      for (int u = pair; u < units; u += npairs) {
        const int nchunks = (nk + chunk - 1) / chunk;
        for (int c = 0; c < nchunks; ++c, ++gc) {
          const int buf = gc & 1;
          if (gc >= 2) mbar_wait_cluster(&acc_empty[buf], ((gc >> 1) - 1) & 1);
          if (gc < 16) pstamp(p, 16 + gc);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t tmem_d = tmem_base + (uint32_t)(buf * BN);
          const int kb_beg = c * chunk, kb_end = min(nk, kb_beg + chunk);
          for (int kb = kb_beg; kb < kb_end; ++kb, ++g) {
            const int s = g % STAGES;
            mbar_wait_cluster(&ready[s], (g / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t a0 = smem_u32(tile(s, 0)), a1 = smem_u32(tile(s, 1));
            const uint32_t b0 = smem_u32(tile(s, 2)), b1 = smem_u32(tile(s, 3));
            const uint64_t a_hi = amn ? smem_desc_mn_sw128(a0) : smem_desc_sw128(a0);
            const uint64_t a_lo = amn ? smem_desc_mn_sw128(a1) : smem_desc_sw128(a1);
            const uint64_t b_hi = bmn ? smem_desc_mn_sw128(b0) : smem_desc_sw128(b0);
            const uint64_t b_lo = bmn ? smem_desc_mn_sw128(b1) : smem_desc_sw128(b1);
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t da = astep * k, db = bstep * k;
              const uint32_t acc = (kb > kb_beg || k > 0) ? 1u : 0u;
              mma_tf32_pair(tmem_d, a_hi + da, b_hi + db, p.idesc, acc);
              mma_tf32_pair(tmem_d, a_hi + da, b_lo + db, p.idesc, 1u);
              mma_tf32_pair(tmem_d, a_lo + da, b_hi + db, p.idesc, 1u);
              // both operands raw: hi = trunc_tf32 on both sides makes the
              // dropped lo*lo term sign-biased, so it is kept
              if (lo_lo) mma_tf32_pair(tmem_d, a_lo + da, b_lo + db, p.idesc, 1u);
            }
            if (g == 0) pstamp(p, 3);
            mma_commit_pair(&empty[s]);
          }
          mma_commit_pair(&acc_full[buf]);
          if (gc < 16) pstamp(p, 32 + gc);
        }
      }
    }
    __syncwarp();
  } else if (SINGLE && warp >= 2 + EPI_WARPS) {
    // ---- split warps (TMEM-resident mode): raw stages -> lo planes, then
    // one `ready` arrival per CTA on the leader
    const int st_ = threadIdx.x - 32 * (2 + EPI_WARPS);
    const bool split_a = p.a_mode != kPreSplit, split_b = p.b_mode != kPreSplit;
    int g = 0;
    for (int u = pair; u < units; u += npairs) {
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % STAGES;
        mbar_wait(&full[s], (g / STAGES) & 1);
        if (split_a)
          split_tf32_smem(smem_u32(tile(s, 0)), smem_u32(tile(s, 1)), A_BYTES / 16, st_,
                          32 * SPLIT_WARPS);
        if (split_b)
          split_tf32_smem(smem_u32(tile(s, 2)), smem_u32(tile(s, 3)), C::B_BYTES / 16, st_,
                          32 * SPLIT_WARPS);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_bar(2, 32 * SPLIT_WARPS);
        if (st_ == 0 && kb == nk - 1 && g / nk < 16) pstamp(p, 64 + g / nk);
        if (st_ == 0) {
          if (rank == 0) mbar_arrive(&ready[s]);
          else mbar_arrive_remote(&ready[s], 0);
        }
      }
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;
    float* stage0 = staging + (warp - 2) * 32 * 32 * C::NSTG;
    int nst = 0;  // staging blocks used (round robin over NSTG)
    const bool split_a = p.a_mode != kPreSplit, split_b = p.b_mode != kPreSplit;
    int gc = 0, gs = 0;
    auto split_stage = [&]() {
      const int s = gs % STAGES;
      mbar_wait(&full[s], (gs / STAGES) & 1);
      if (split_a) split_tf32_smem(smem_u32(tile(s, 0)), smem_u32(tile(s, 1)), A_BYTES / 16, et, 256);
      if (split_b)
        split_tf32_smem(smem_u32(tile(s, 2)), smem_u32(tile(s, 3)), C::B_BYTES / 16, et, 256);
      // one arrive per CTA: the 8 warps meet on a named barrier first (a
      // cluster-scope release per warp costs a GPU-wide membar each)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar(1, 32 * EPI_WARPS);
      if (et == 0) {
        if (rank == 0) mbar_arrive(&ready[s]);
        else mbar_arrive_remote(&ready[s], 0);
      }
      ++gs;
    };
    // one finished 32x32 block (this warp's 32 rows x 32 columns from col0):
    // alpha, bias/act epilogue, then a TMA store of the XOR-swizzled staging
    // block or (strided / accumulating C) 4-row x 128-byte stores through it
    auto emit32 = [&](const float* vals, int bz, int row0, int col0, float alpha) {
      const int grow = row0 + lane;
      float* stage = stage0 + 32 * 32 * (nst++ % C::NSTG);
      if (p.tma_store) {
        // the block's previous store has finished reading it (NSTG - 1 may be in flight)
        if (lane == 0) {
          if (C::NSTG == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 v = make_float4(vals[4 * q] * alpha, vals[4 * q + 1] * alpha,
                                 vals[4 * q + 2] * alpha, vals[4 * q + 3] * alpha);
          if (grow < p.M) epi4(p, bz, grow, col0 + 4 * q, v);
          *reinterpret_cast<float4*>(stage + lane * 32 + 4 * (q ^ (lane & 7))) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&map_c, stage, col0, row0, bz);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        return;
      }
      float* cbase = p.C + bz * p.scb;
      const int sub_r = lane >> 3, sub_c = (lane & 7) * 4;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stage + lane * 32 + 4 * (q ^ (lane & 7))) =
            make_float4(vals[4 * q] * alpha, vals[4 * q + 1] * alpha, vals[4 * q + 2] * alpha,
                        vals[4 * q + 3] * alpha);
      __syncwarp();
      const int col = col0 + sub_c;
#pragma unroll 4
      for (int i = 0; i < 32; i += 4) {
        const int row = row0 + i + sub_r;
        const int srow = i + sub_r;
        float4 v = *reinterpret_cast<const float4*>(stage + srow * 32 +
                                                    4 * ((sub_c >> 2) ^ (srow & 7)));
        if (row < p.M && col < p.N) {
          float* q = cbase + (int64_t)row * p.scm + (int64_t)col * p.scn;
          if (p.scn == 1 && col + 3 < p.N && ((reinterpret_cast<uintptr_t>(q) & 15) == 0)) {
            if (p.accumulate) {
              const float4 o = *reinterpret_cast<const float4*>(q);
              v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
            }
            epi4(p, bz, row, col, v);
            *reinterpret_cast<float4*>(q) = v;
          } else {
            if (p.accumulate) {
              if (col < p.N) v.x += q[0];
              if (col + 1 < p.N) v.y += q[p.scn];
              if (col + 2 < p.N) v.z += q[2 * p.scn];
              if (col + 3 < p.N) v.w += q[3 * p.scn];
            }
            epi4(p, bz, row, col, v);
            const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (col + j < p.N) q[(int64_t)j * p.scn] = e[j];
          }
        }
      }
      __syncwarp();
    };
    auto release = [&](int buf) {
      asm volatile("tcgen05.fence::before_thread_sync;");
      named_bar(1, 32 * EPI_WARPS);
      if (et == 0) {
        if (rank == 0) mbar_arrive(&acc_empty[buf]);
        else mbar_arrive_remote(&acc_empty[buf], 0);
      }
    };
    auto tile_of = [&](int u, int* bz, int* m0, int* n0) {
      *bz = u / tiles_per_batch;
      const int r = u % tiles_per_batch;
      *m0 = (r / p.ntn) * 256 + (int)rank * 128;
      *n0 = (r % p.ntn) * BN;
    };
    auto alpha_of = [&](int bz, int grow) {
      return (p.alpha_rows && grow < p.M) ? __ldg(p.alpha_rows + (int64_t)bz * p.M + grow) : 1.f;
    };
    if constexpr (SINGLE) {
      // the whole K accumulates in TMEM (short K): each finished tile streams
      // TMEM -> registers (32 columns at a time) -> store; no register
      // accumulator, so 256-wide tiles fit.  The drain of tile t runs while
      // the MMA works on tile t+1 (its stages are split first).
      auto drain_store = [&](int u) {
        int bz, m0, n0;
        tile_of(u, &bz, &m0, &n0);
        const int buf = gc & 1;
        mbar_wait(&acc_full[buf], (gc >> 1) & 1);
        if (et == 0 && gc < 16) pstamp(p, 48 + gc);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int row0 = m0 + quarter * 32;
        const float alpha = alpha_of(bz, row0 + lane);
#pragma unroll 1
        for (int cc = 0; cc < EPI_COLS; cc += 32) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) +
                        (uint32_t)(buf * BN + half * EPI_COLS + cc), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
          if (cc + 32 >= EPI_COLS) release(buf);  // all of this buffer is in registers
          emit32(f, bz, row0, n0 + half * EPI_COLS + cc, alpha);
        }
        if (et == 0 && gc < 8) pstamp(p, 4 + gc);
        ++gc;
      };
      for (int u = pair; u < units; u += npairs) drain_store(u);
    } else {
      float acc[EPI_COLS];
      auto drain = [&]() {
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
        release(buf);
        ++gc;
      };
      for (int u = pair; u < units; u += npairs) {
        int bz, m0, n0;
        tile_of(u, &bz, &m0, &n0);
        const int nchunks = (nk + chunk - 1) / chunk;
#pragma unroll
        for (int j = 0; j < EPI_COLS; ++j) acc[j] = 0.f;
        for (int c = 0; c < nchunks; ++c) {
          const int kb_beg = c * chunk, kb_end = min(nk, kb_beg + chunk);
          for (int kb = kb_beg; kb < kb_end; ++kb) split_stage();
          if (c > 0) drain();
        }
        drain();
        const int row0 = m0 + quarter * 32;
        const float alpha = alpha_of(bz, row0 + lane);
#pragma unroll
        for (int cc = 0; cc < EPI_COLS; cc += 32)
          emit32(&acc[cc], bz, row0, n0 + half * EPI_COLS + cc, alpha);
      }
    }
    if (p.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) pstamp(p, 12);
  cluster_sync_all();  // no CTA leaves while its peer may still arrive on its barriers
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// ---- host ----

static int64_t align_up(int64_t x) { return (x + 255) / 256 * 256; }

static bool plane_map(CUtensorMap* map, const float* base, int64_t Kp, int64_t rows, int64_t batch,
                      int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(Kp * 4), (cuuint64_t)(rows * Kp * 4)};
  cuuint32_t box[3] = {BK, (cuuint32_t)box_rows, 1};
  return encode(map, base, dims, strides, box);
}

static int raw_mode(const float* base, int64_t rows, int64_t K, int64_t nb, int64_t sb, int64_t sr,
                    int64_t sk) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return kPreSplit;
  const bool b_ok = nb == 1 || ((sb * 4) % 16 == 0 && sb > 0);
  if (!b_ok) return kPreSplit;
  if (sk == 1 && (rows == 1 || ((sr * 4) % 16 == 0 && sr >= K))) return kRawK;
  if (sr == 1 && rows > 1 && (sk * 4) % 16 == 0 && sk >= rows) return kRawMN;
  return kPreSplit;
}

static bool raw_map(CUtensorMap* map, int mode, const float* base, int64_t rows, int64_t K,
                    int64_t nb, int64_t sb, int64_t sr, int64_t sk, int box_rows) {
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

static int num_pairs() {
  static int n = 0;
  if (!n) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    n = std::max(1, (sms > 0 ? sms : kNumSMs) / 2);
  }
  return n;
}

// N tile: the smaller of (waves x tile width), ties to 256 (less operand traffic)
// 256-wide tiles only in the TMEM-resident (short-K) mode: with register
// accumulation a 128 x 256 half tile needs 128 accumulators per epilogue
// thread, more than 10 warps per SM can hold
static int choose_bn(const GemmArgs& g, bool single) {
  if (const char* e = getenv("PFB_PAIR_BN")) return (atoi(e) == 256 && single) ? 256 : 128;
  if (g.N <= 128 || !single) return 128;
  const int64_t ntm = (g.M + 255) / 256;
  auto cost = [&](int bn) {
    const int64_t units = ntm * ((g.N + bn - 1) / bn) * g.batch;
    return (double)((units + num_pairs() - 1) / num_pairs()) * bn;
  };
  return cost(256) <= cost(128) ? 256 : 128;
}

static int pair_chunk() {
  static const int c = [] {
    const char* e = getenv("PFB_PAIR_CHUNK");
    const int v = e ? atoi(e) : 4;
    return v >= 1 && v <= 64 ? v : 4;
  }();
  return c;
}

template <int BN, bool SINGLE>
static int launch_pair(const CUtensorMap& mah, const CUtensorMap& mal, const CUtensorMap& mbh,
                       const CUtensorMap& mbl, const CUtensorMap& mc, const PParams& p,
                       cudaStream_t s) {
  using C = Cfg<BN, SINGLE>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pair_kernel<BN, SINGLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM);
    attr = true;
  }
  const int64_t units = (int64_t)p.ntm * p.ntn * p.batch;
  const int pairs = (int)std::min<int64_t>(units, num_pairs());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(threads_of<SINGLE>());
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  kernel_launches()++;
  cudaLaunchKernelEx(&cfg, pair_kernel<BN, SINGLE>, mah, mal, mbh, mbl, mc, p);
  return launch_status();
}

}  // namespace tcp

int gemm_tcgen05_pair(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s, int variant) {
  using namespace tcp;
  if (!gemm_tcgen05_eligible(g) || g.M <= 128) return PFB_E_UNSUPPORTED;
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int a_bc = g.sab == 0 && g.batch > 1;
  const int b_bc = g.sbb == 0 && g.batch > 1 && !(g.kscale && g.skb != 0);
  const int64_t ba = a_bc ? 1 : g.batch, bb = b_bc ? 1 : g.batch;
  // short K: the whole accumulation stays in TMEM (error ~K/4096 x 1e-4
  // relative from the tensor core's truncating accumulation, measured)
  const int64_t Kp0 = (g.K + 3) / 4 * 4;
  const bool single = Kp0 <= 256 && !getenv_flag("PFB_PAIR_NO_SINGLE");
  const int bn = choose_bn(g, single);
  const int bnh = bn / 2;
  int am = kPreSplit, bm = kPreSplit;
  if (variant == 2) {
    am = raw_mode(g.A, g.M, g.K, ba, g.sab, g.sam, g.sak);
    bm = g.kscale ? kPreSplit : raw_mode(g.B, g.N, g.K, bb, g.sbb, g.sbn, g.sbk);
    if (bm == kRawMN && bnh % 32 != 0) bm = kPreSplit;
  }
  const int64_t need = (am == kPreSplit ? 2 * align_up(ba * g.M * Kp * 4) : 0) +
                       (bm == kPreSplit ? 2 * align_up(bb * g.N * Kp * 4) : 0);
  if (need > 0 && (ws == nullptr || ws_bytes < need)) return PFB_E_UNSUPPORTED;
  char* w = static_cast<char*>(ws);
  CUtensorMap mah, mal, mbh, mbl;
  if (am == kPreSplit) {
    float* ah = reinterpret_cast<float*>(w); w += align_up(ba * g.M * Kp * 4);
    float* al = reinterpret_cast<float*>(w); w += align_up(ba * g.M * Kp * 4);
    tc_split_launch(g.A, ba, g.M, g.K, Kp, g.sab, g.sam, g.sak, ah, al, nullptr, 0, 0, s);
    if (!plane_map(&mah, ah, Kp, g.M, ba, 128) || !plane_map(&mal, al, Kp, g.M, ba, 128))
      return PFB_E_UNSUPPORTED;
  } else {
    if (!raw_map(&mah, am, g.A, g.M, g.K, ba, g.sab, g.sam, g.sak, 128)) return PFB_E_UNSUPPORTED;
    mal = mah;
  }
  if (bm == kPreSplit) {
    float* bh = reinterpret_cast<float*>(w); w += align_up(bb * g.N * Kp * 4);
    float* bl = reinterpret_cast<float*>(w); w += align_up(bb * g.N * Kp * 4);
    tc_split_launch(g.B, bb, g.N, g.K, Kp, g.sbb, g.sbn, g.sbk, bh, bl, g.kscale, g.skb, g.skk, s);
    if (!plane_map(&mbh, bh, Kp, g.N, bb, bnh) || !plane_map(&mbl, bl, Kp, g.N, bb, bnh))
      return PFB_E_UNSUPPORTED;
  } else {
    if (!raw_map(&mbh, bm, g.B, g.N, g.K, bb, g.sbb, g.sbn, g.sbk, bnh)) return PFB_E_UNSUPPORTED;
    mbl = mbh;
  }
  CUtensorMap mc = mah;
  int tma_store = 0;
  if (!g.accumulate && g.scn == 1 && (g.N == 1 || (g.scm * 4) % 16 == 0) &&
      (g.batch == 1 || (g.scb * 4) % 16 == 0) && (reinterpret_cast<uintptr_t>(g.C) & 15) == 0 &&
      !getenv_flag("PFB_NO_TMA_STORE")) {
    const int64_t ldc = g.M == 1 ? (g.N + 3) / 4 * 4 : g.scm;
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)g.batch};
    cuuint64_t strides[2] = {(cuuint64_t)(ldc * 4),
                             (cuuint64_t)((g.batch == 1 ? ldc * g.M : g.scb) * 4)};
    cuuint32_t box[3] = {32, 32, 1};
    tma_store = encode(&mc, g.C, dims, strides, box) ? 1 : 0;
  }
  // kind::tf32, D=f32, M=256 (pair), N=bn; bits 15/16: A/B MN-major
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(am == kRawMN) << 15) |
                         ((uint32_t)(bm == kRawMN) << 16) | ((uint32_t)(bn >> 3) << 17) |
                         ((uint32_t)(256 >> 4) << 24);
  PParams p{(int)g.M, (int)g.N, (int)Kp, (int)g.batch,
            (int)((g.M + 255) / 256), (int)((g.N + bn - 1) / bn), a_bc, b_bc, am, bm, idesc,
            g.C, g.scb, g.scm, g.scn, g.alpha_rows, g.accumulate,
            g.bias, g.sxb, g.sxm, g.sxn, g.act, tma_store, pair_chunk(), g.dy, g.sdb, g.sdm,
            g.sdn, g.dop, tc_trace_buffer()};
  if (single)
    return bn == 256 ? launch_pair<256, true>(mah, mal, mbh, mbl, mc, p, s)
                     : launch_pair<128, true>(mah, mal, mbh, mbl, mc, p, s);
  return launch_pair<128, false>(mah, mal, mbh, mbl, mc, p, s);
}

}  // namespace pfb
