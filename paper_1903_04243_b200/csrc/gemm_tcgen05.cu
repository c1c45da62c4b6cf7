// tcgen05 / TMEM / TMA GEMM path (3xTF32 for fp32 accuracy) -- placeholder
// until the kernel lands; the SIMT path serves every shape meanwhile.
#include "gemm.cuh"

namespace pfb {
bool gemm_tcgen05_eligible(const GemmArgs&) { return false; }
int gemm_tcgen05(const GemmArgs&, cudaStream_t) { return PFB_E_UNSUPPORTED; }
}  // namespace pfb
