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
};

int gemm_simt(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s);
int64_t gemm_simt_workspace(const GemmArgs& g);
// returns PFB_E_UNSUPPORTED when the shape/layout is not eligible
int gemm_tcgen05(const GemmArgs& g, void* ws, int64_t ws_bytes, cudaStream_t s);
int64_t gemm_tcgen05_workspace(const GemmArgs& g);
bool gemm_tcgen05_eligible(const GemmArgs& g);    // layout constraints
bool gemm_tcgen05_profitable(const GemmArgs& g);  // size heuristic for auto

}  // namespace pfb
