// SIMT fp32 GEMM for shapes the tensor-core path does not take: tiny M/N/K
// (per-example conv filter grads 9x8, K=1 outer products, K=10 cotangents),
// odd strides and ragged batches.  64x64x16 tiles, 256 threads, 4x4 register
// micro-tile; operands staged through shared memory with the global read
// mapped onto whichever of their two strides is unit (coalesced for both
// normal and transposed views).  Exact fp32 FMA accumulation.
#include "gemm.cuh"

namespace pfb {

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int64_t b = blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const float* A = g.A + b * g.sab;
  const float* B = g.B + b * g.sbb;
  const int tid = threadIdx.x;
  const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
  float acc[4][4] = {};
  const bool a_kfast = g.sak == 1 || g.sam != 1;
  const bool b_nfast = g.sbn == 1 || g.sbk != 1;
  for (int64_t k0 = 0; k0 < g.K; k0 += BK) {
    // A tile: BM x BK = 1024 elements, 4 per thread
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int e = tid + j * 256;
      int mm, kk;
      if (a_kfast) { mm = e / BK; kk = e % BK; } else { kk = e / BM; mm = e % BM; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < g.M && gk < g.K) ? __ldg(A + gm * g.sam + gk * g.sak) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int e = tid + j * 256;
      int kk, nn;
      if (b_nfast) { kk = e / BN; nn = e % BN; } else { nn = e / BK; kk = e % BK; }
      int64_t gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < g.K && gn < g.N) ? __ldg(B + gk * g.sbk + gn * g.sbn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tm + i];
#pragma unroll
      for (int i = 0; i < 4; ++i) bb[i] = Bs[kk][tn + i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* C = g.C + b * g.scb;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gm = m0 + tm + i;
    if (gm >= g.M) continue;
    float alpha = g.alpha_rows ? g.alpha_rows[b * g.M + gm] : 1.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t gn = n0 + tn + j;
      if (gn >= g.N) continue;
      float* p = C + gm * g.scm + gn * g.scn;
      float v = acc[i][j] * alpha;
      *p = g.accumulate ? *p + v : v;
    }
  }
}

// Tiny-K kernel (K <= 32): outer-product-like, one thread per output element,
// operands read straight from global (L1/L2 resident rows).  Store-bound.
__global__ void __launch_bounds__(256) gemm_smallk_kernel(GemmArgs g) {
  const int64_t total = g.batch * g.M * g.N;
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < total;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = lin % g.N;
    int64_t t = lin / g.N;
    int64_t m = t % g.M;
    int64_t b = t / g.M;
    const float* a = g.A + b * g.sab + m * g.sam;
    const float* bb = g.B + b * g.sbb + n * g.sbn;
    float acc = 0.f;
    for (int64_t k = 0; k < g.K; ++k) acc = fmaf(__ldg(a + k * g.sak), __ldg(bb + k * g.sbk), acc);
    if (g.alpha_rows) acc *= g.alpha_rows[b * g.M + m];
    float* p = g.C + b * g.scb + m * g.scm + n * g.scn;
    *p = g.accumulate ? *p + acc : acc;
  }
}

int gemm_simt(const GemmArgs& g, cudaStream_t s) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return 0;
  if (g.K <= 8) {
    gemm_smallk_kernel<<<grid_for(g.batch * g.M * g.N, 256), 256, 0, s>>>(g);
    return launch_status();
  }
  dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM), (unsigned)g.batch);
  if (grid.y > 65535 || grid.z > 65535) {
    // fall back to the grid-stride small-K kernel for extreme shapes
    gemm_smallk_kernel<<<grid_for(g.batch * g.M * g.N, 256), 256, 0, s>>>(g);
    return launch_status();
  }
  gemm_simt_kernel<<<grid, 256, 0, s>>>(g);
  return launch_status();
}

}  // namespace pfb
