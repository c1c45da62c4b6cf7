// Fused elementwise register programs (pass F3): the program encoding shared
// by the interpreter kernels (elementwise.cu) and the specialising compiler
// (fused_jit.cu).
#pragma once
#include "common.cuh"

namespace pfb {

constexpr int kMaxSteps = 48;
constexpr int kMaxRegs = 16;
enum FusedOpc { F_LOAD = 64, F_CONST = 65, F_SELECT = 68 };

constexpr int kMaxOuts = 8;
struct FusedProgram {
  int n_in, n_steps;
  int in_dtype[8];
  int code[kMaxSteps][4];  // opcode, dst, src1, src2 (src1 = input / const bits)
  int n_out;               // outputs: registers stored after the program
  int out_reg[kMaxOuts];
  int out_dt[kMaxOuts];    // PFB_F32 or PFB_BOOL
};

struct FusedOuts {
  void* p[kMaxOuts];
};

// Launch `P` as a kernel specialised to it (straight-line code, registers
// in registers); false when the specialiser is unavailable or declines
// (the caller then runs the interpreter kernel).  V, modes, ngroups, idx64
// as for the interpreter launch.
bool fused_jit_launch(const FusedProgram& P, int V, bool idx64, uint32_t modes, const Layout& L,
                      int64_t ngroups, const FusedOuts& outs, const void* const* p,
                      cudaStream_t s);

// the same for an integer-domain program (fused_int_kernel), one element per
// thread
bool fused_int_jit_launch(const FusedProgram& P, bool idx64, const Layout& L, int64_t n,
                          const FusedOuts& outs, const void* const* p, cudaStream_t s);

}  // namespace pfb
