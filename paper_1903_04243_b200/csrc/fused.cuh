// Fused elementwise register programs (pass F3): the program encoding shared
// by the interpreter kernels (elementwise.cu) and the specialising compiler
// (fused_jit.cu).
#pragma once
#include "common.cuh"

namespace pfb {

constexpr int kMaxSteps = 96;
constexpr int kMaxRegs = 32;
constexpr int kMaxIn = kMaxFOps - 1;  // 16 tensor inputs
enum FusedOpc { F_LOAD = 64, F_CONST = 65, F_SELECT = 68 };

constexpr int kMaxOuts = 12;
struct FusedProgram {
  int n_in, n_steps;
  int in_dtype[kMaxIn];
  int code[kMaxSteps][4];  // opcode, dst, src1, src2 (src1 = input / const bits)
  int n_out;               // outputs: registers stored after the program
  int out_reg[kMaxOuts];
  int out_dt[kMaxOuts];    // PFB_F32 or PFB_BOOL
};

struct FusedOuts {
  void* p[kMaxOuts];
};

struct FusedIns {
  const void* p[kMaxIn];
};

// per-operand feed modes, 2 bits each (operand 0 = the outputs): 0 = 128-bit
// vector, 1 = stride-0 broadcast, 2 = strided scalar
using FeedModes = uint64_t;

// Split-K partial-sum inputs (pass F15): input k is the sum of S[k] copies
// at element offsets j * st[k] (j = 0..S[k]-1, summed left to right as
// loaded); S[k] <= 1 = a plain input.  Only the specialised kernels take them.
constexpr int kMaxParts = 32;
struct PartsSpec {
  int S[kMaxIn];
  int64_t st[kMaxIn];
  bool any() const {
    for (int k = 0; k < kMaxIn; ++k)
      if (S[k] > 1) return true;
    return false;
  }
};

// Launch `P` as a kernel specialised to it (straight-line code, registers
// in registers); false when the specialiser is unavailable or declines
// (the caller then runs the interpreter kernel).  V, modes, ngroups, idx64
// as for the interpreter launch.
bool fused_jit_launch(const FusedProgram& P, int V, bool idx64, FeedModes modes, const FLayout& L,
                      int64_t ngroups, const FusedOuts& outs, const FusedIns& ins,
                      cudaStream_t s, const PartsSpec* parts = nullptr);

// Row-sum feeds (pass F16): rowsum[k] >= 0 makes input k the sum of input
// rowsum[k] (after its partials) over the layout's innermost dim, computed in
// the kernel (one row per block); false when the shape does not fit (the
// caller then materialises the sums).  V = 1, specialised kernels only.
bool fused_rows_jit_launch(const FusedProgram& P, FeedModes modes, const FLayout& L, int64_t n,
                           const FusedOuts& outs, const FusedIns& ins, cudaStream_t s,
                           const PartsSpec* parts, const int* rowsum);

// the same for an integer-domain program (fused_int_kernel), one element per
// thread
bool fused_int_jit_launch(const FusedProgram& P, bool idx64, const FLayout& L, int64_t n,
                          const FusedOuts& outs, const FusedIns& ins, cudaStream_t s);

}  // namespace pfb
