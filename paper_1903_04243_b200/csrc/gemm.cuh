// Internal GEMM interface shared by the SIMT and tcgen05 paths.
#pragma once
#include "common.cuh"

namespace pfb {

// C[b] (M x N) = A[b] (M x K) * B[b] (K x N), all fp32; strides in elements.
struct GemmArgs {
  int64_t batch, M, N, K;
  const float* A;
  int64_t sab, sam, sak;
  const float* B;
  int64_t sbb, sbk, sbn;
  float* C;
  int64_t scb, scm, scn;
  const float* alpha_rows;  // nullable: C[m, :] *= alpha_rows[b*M + m]
  int accumulate;           // C += result
  // fused prologue / epilogue (passes.fuse_matmul_epilogues):
  //   C = act(alpha * (A diag(kscale) B) [+ C] + bias)
  const float* kscale = nullptr;  // nullable, per (batch, k): scales B's rows
  int64_t skb = 0, skk = 0;
  const float* bias = nullptr;    // nullable, broadcast to (batch, M, N) by strides
  int64_t sxb = 0, sxm = 0, sxn = 0;
  int act = 0;                    // PFB_ACT_*
  // derivative epilogue (autodiff's tanh'/sigmoid' cotangent multiply):
  //   C *= (1 - y^2)  [PFB_DOP_DTANH]   or   C *= y (1 - y)  [PFB_DOP_DSIGMOID]
  const float* dy = nullptr;      // y, broadcast to (batch, M, N) by strides
  int64_t sdb = 0, sdm = 0, sdn = 0;
  int dop = 0;
  // nullable: B's dense K-major tf32 hi / lo planes [bb][N][Kp], made once by
  // pfb_gemm_split_planes for a loop-invariant weight (the executor caches
  // them per constant); the tcgen05 path then reads B with no split at all
  // and needs 3 products (B's RN split keeps the dropped lo*lo term unbiased)
  const float* b_hi = nullptr;
  const float* b_lo = nullptr;
  __host__ __device__ bool has_epi() const { return bias != nullptr || act != 0 || dop != 0; }
};

// the derivative factor of the epilogue at (b, m, n)
__device__ __forceinline__ float dop_factor(int dop, const float* dy, int64_t off) {
  const float y = __ldg(dy + off);
  return dop == PFB_DOP_DTANH ? 1.f - y * y : y * (1.f - y);
}

__device__ __forceinline__ float apply_act(int act, float v) {
  switch (act) {
    case PFB_ACT_TANH: return tanhf(v);
    case PFB_ACT_SIGMOID: return 1.f / (1.f + expf(-v));
    case PFB_ACT_RELU: return v != v ? v : (v >= 0.f ? v : 0.f);
    default: return v;
  }
}

// bias + activation on a finished output value
__device__ __forceinline__ float epi_value(const GemmArgs& g, int64_t b, int64_t m, int64_t n,
                                           float v) {
  if (g.bias) v += __ldg(g.bias + b * g.sxb + m * g.sxm + n * g.sxn);
  v = apply_act(g.act, v);
  if (g.dop) v *= dop_factor(g.dop, g.dy, b * g.sdb + m * g.sdm + n * g.sdn);
  return v;
}

__device__ __forceinline__ float kscale_at(const GemmArgs& g, int64_t b, int64_t k) {
  return g.kscale ? __ldg(g.kscale + b * g.skb + k * g.skk) : 1.f;
}

int gemm_simt(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s);
int gemm_simt_v(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s, int splits_want,
                bool ws_reduce);
bool gemm_simt_splittable(const GemmArgs& g);
int64_t gemm_simt_workspace_max(const GemmArgs& g);
int64_t gemm_simt_workspace(const GemmArgs& g);
// returns PFB_E_UNSUPPORTED when the shape/layout is not eligible
// variant: 0 = auto, 1 = operands pre-split by split_kernel, 2 = raw operands
// fed by TMA and split in shared memory wherever the layout allows it
// ksplit_want > 0 forces that many k-splits (autotune candidates), 0 = model
// bn: tile width (MMA N) 128, 64 or 32 (skinny-M problems: more CTAs over N)
int gemm_tcgen05(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s, int variant = 0,
                 int ksplit_want = 0, int bn = 128);
int64_t gemm_tcgen05_workspace(const GemmArgs& g);
// C = epi(A1 B1 + A2 B2) in one tcgen05 launch (consecutive K ranges of one
// accumulation); g1 carries C and the epilogue, g2 only its operands
int gemm_tcgen05_dual(const GemmArgs& g1, const GemmArgs& g2, void* ws, int64_t ws_bytes,
                      cudaStream_t s, int variant = 0, int ksplit_want = 0, int bn = 128);
int64_t gemm_tcgen05_dual_workspace(const GemmArgs& g1, const GemmArgs& g2);
// PFB_TC_TRACE=1: 16-slot globaltimer stamp buffer (device), else nullptr
unsigned long long* tc_trace_buffer();
bool gemm_tcgen05_eligible(const GemmArgs& g);    // layout constraints
bool gemm_tcgen05_raw_possible(const GemmArgs& g);
bool gemm_tcgen05_profitable(const GemmArgs& g);  // size heuristic for auto
// CTA-pair (cta_group::2) kernel: 256-row pair tiles, N tile 128 or 256;
// variant 1 = pre-split planes, 2 = raw TMA feed where the layout allows it
int gemm_tcgen05_pair(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s, int variant);
// split-K partials GEMM (gemm_parts.cu): S k-splits of a batch-1 GEMM written
// to parts + s*part_stride (row stride ldc), bias in split 0, no reduction
// g2 (nullable): a dual GEMM's second operand pair (parts = sums over both K ranges)
int gemm_parts_count(const GemmArgs& g, const GemmArgs* g2 = nullptr);  // S (0: not applicable)
int64_t gemm_parts_workspace(const GemmArgs& g, const GemmArgs* g2 = nullptr);
int gemm_parts(const GemmArgs& g, const GemmArgs* g2, int S, float* parts, int64_t part_stride,
               int64_t ldc, void* ws, int64_t ws_bytes, cudaStream_t s);
// dense K-major hi/lo tf32 planes [batch][rows][Kp] of an operand view
int64_t gemm_planes_bytes(const GemmArgs& g);  // both planes of B (0: not splittable)
void tc_split_launch(const float* x, int64_t batch, int64_t rows, int64_t K, int64_t Kp, int64_t sb,
                     int64_t sr, int64_t sk, float* hi, float* lo, const float* kscale,
                     int64_t skb, int64_t skk, cudaStream_t s);

}  // namespace pfb
