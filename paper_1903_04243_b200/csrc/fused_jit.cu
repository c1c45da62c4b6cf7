// Specialising compiler for fused elementwise programs (pass F3 groups).
//
// The interpreter kernel (elementwise.cu fused_kernel) keeps the program's
// register file in local memory and dispatches every step through a switch:
// at HBM-scale tensors it is L1/issue bound (~30% of HBM on a 6-step chain,
// profiles/r01/membw_b200.json), and at small sizes its per-step local-memory
// round trips are the launch's latency.  For every group (PFB_JIT_MIN sets a
// size floor) this file emits the program as straight-line CUDA C++ -- one
// SSA value per
// step and lane, the input feed modes and dtypes baked in, the same float
// expressions the interpreter evaluates (np_max/np_min NaN rules, IEEE div,
// expf/logf/tanhf), compiled with -fmad=false so no step is contracted into
// an FMA the interpreter would not perform -- compiles it once with NVRTC for
// sm_100a and caches the kernel per (program, feed modes, width, device).
// Results are therefore the interpreter's, bit for bit; tests/test_gpu_jit.py
// checks exactly that.
//
// NVRTC is dlopen'ed (no link-time dependency); without it, or with
// PFB_NO_JIT=1, every group runs on the interpreter.  Module loads made while
// a stream is being captured switch the thread to relaxed capture mode for
// the load only.
#include "fused.cuh"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

namespace pfb {
namespace {

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  bool ok = false;
};

struct Driver {
  decltype(&cuModuleLoadData) load = nullptr;
  decltype(&cuModuleGetFunction) get = nullptr;
  decltype(&cuLaunchKernelEx) launch = nullptr;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    const char* names[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return r;
    r.create = (decltype(r.create))dlsym(h, "nvrtcCreateProgram");
    r.compile = (decltype(r.compile))dlsym(h, "nvrtcCompileProgram");
    r.log_size = (decltype(r.log_size))dlsym(h, "nvrtcGetProgramLogSize");
    r.log = (decltype(r.log))dlsym(h, "nvrtcGetProgramLog");
    r.cubin_size = (decltype(r.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    r.cubin = (decltype(r.cubin))dlsym(h, "nvrtcGetCUBIN");
    r.destroy = (decltype(r.destroy))dlsym(h, "nvrtcDestroyProgram");
    r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
    return r;
  }();
  return n;
}

template <typename F>
bool entry(const char* name, F* out) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *out = reinterpret_cast<F>(p);
  return true;
}

const Driver& driver() {
  static Driver d = [] {
    Driver r;
    r.ok = entry("cuModuleLoadData", &r.load) && entry("cuModuleGetFunction", &r.get) &&
           entry("cuLaunchKernelEx", &r.launch);
    return r;
  }();
  return d;
}

// ---------------------------------------------------------------------------
// source generation

const char* kPrelude = R"(
typedef long long i64;
struct Layout { int rank; int nops; i64 shape[%d]; i64 st[%d][%d]; };
struct Outs { void* p[%d]; };
struct Ins { const void* p[%d]; };
__device__ __forceinline__ float np_max(float a, float b) {
  return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b));
}
__device__ __forceinline__ float np_min(float a, float b) {
  return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b));
}
)";

std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

// Offsets of every operand for group index g, straight-line with the
// layout's shape and strides as literals (divisions by constants, zero-stride
// terms dropped, 32-bit arithmetic when every offset fits): the generic loop
// over the layout's dims costs ~10 instructions per operand and dim, which
// dominated small many-input groups (the LSTM cell: 19 operands x 3 dims).
std::string gen_offsets(const FLayout& L, int nops, int V, bool idx64, bool off32, int lpr = 0) {
  std::string s;
  const char* IT = idx64 ? "i64" : "unsigned";
  const char* OT = off32 ? "int" : "i64";
  if (lpr > 0) {  // short rows (F16): lanes [lpr*r, lpr*r + W) of a warp hold row r
    const long long W = (long long)L.shape[L.rank - 1];
    long long R = 1;
    for (int d = 0; d < L.rank - 1; ++d) R *= (long long)L.shape[d];
    s += fmt("    const %s rw_r = g / %d, rw_c = g %% %d;\n", IT, lpr, lpr);
    s += fmt("    const bool valid = rw_c < %lld && rw_r < %lld;\n", W, R);
    s += fmt("    %s lin = valid ? rw_r * %lld + rw_c : 0;\n", IT, W);
  } else {
    s += fmt("    %s lin = g * %d;\n", IT, V);
  }
  std::string terms[kMaxFOps];
  for (int d = L.rank - 1; d >= 0; --d) {
    std::string c;
    if (d == 0) {
      c = "lin";
    } else {
      s += fmt("    const %s c%d = lin %% (%s)%lld; lin /= (%s)%lld;\n", IT, d, IT,
               (long long)L.shape[d], IT, (long long)L.shape[d]);
      c = fmt("c%d", d);
    }
    for (int o = 0; o < nops; ++o) {
      const long long st = (long long)L.st[o][d];
      if (st == 0) continue;
      std::string t = st == 1 ? fmt("(%s)%s", OT, c.c_str())
                              : fmt("(%s)%s * (%s)%lld", OT, c.c_str(), OT, st);
      terms[o] += (terms[o].empty() ? "" : " + ") + t;
    }
  }
  s += fmt("    i64 off[%d];\n", nops);
  for (int o = 0; o < nops; ++o)
    s += fmt("    off[%d] = (i64)(%s);\n", o, terms[o].empty() ? "0" : terms[o].c_str());
  return s;
}

// a unary program opcode (16 + PFB_*) applied to expression x, as the
// program steps evaluate it; op 0 = x itself
std::string unary_expr(int op, const std::string& x) {
  switch (op) {
    case 0: return x;
    case 16 + PFB_NEG: return "(-" + x + ")";
    case 16 + PFB_EXP: return "expf(" + x + ")";
    case 16 + PFB_LOG: return "logf(" + x + ")";
    case 16 + PFB_RELU: return "np_max(" + x + ", 0.f)";
    case 16 + PFB_TANH: return "tanhf(" + x + ")";
    case 16 + PFB_SIGMOID: return "(1.f / (1.f + expf(-" + x + ")))";
    case 16 + PFB_SQUARE: return "(" + x + " * " + x + ")";
    default: return x;
  }
}

std::string gen_source(const FusedProgram& P, int V, bool idx64, FeedModes modes,
                       const PartsSpec* PS = nullptr, const FLayout* LS = nullptr,
                       bool off32 = false, const int* RS = nullptr, int lpr = 0) {
  std::string s = fmt(kPrelude, kMaxRank, kMaxFOps, kMaxRank, kMaxOuts, kMaxIn);
  const char* IT = idx64 ? "i64" : "unsigned";
  const int nops = P.n_in + 1;
  auto nparts = [&](int k) { return (PS && PS->S[k] > 1) ? PS->S[k] : 1; };
  // row-sum feeds: one row per block, blockDim = the row (baked layout)
  const int nthr = (RS && LS && lpr == 0) ? (int)LS->shape[LS->rank - 1] : 256;
  if (PS) {
    s += fmt("struct Parts { i64 st[%d]; };\n", kMaxIn);
    s += fmt("extern \"C\" __global__ void __launch_bounds__(%d) pfb_fused_jit(Layout L, %s ngroups, "
             "Outs outs, Ins ins, Parts PT) {\n", nthr, IT);
  } else {
    s += fmt("extern \"C\" __global__ void __launch_bounds__(%d) pfb_fused_jit(Layout L, %s ngroups, "
             "Outs outs, Ins ins) {\n", nthr, IT);
  }
  s += "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n"
       "  asm volatile(\"griddepcontrol.launch_dependents;\" :::);\n"
       "  const int ir = L.rank - 1;\n";
  s += fmt("  for (%s g = blockIdx.x * (%s)blockDim.x + threadIdx.x; g < ngroups; "
           "g += (%s)gridDim.x * blockDim.x) {\n", IT, IT, IT);
  if (LS) {
    s += gen_offsets(*LS, nops, V, idx64, off32, lpr);
  } else {
    s += fmt("    i64 off[%d];\n", nops);
    s += fmt("    if (L.rank == 1) { for (int o = 0; o < %d; ++o) off[o] = (i64)(g * %d) * L.st[o][0]; }\n",
             nops, V);
    s += fmt("    else { %s lin = g * %d;\n", IT, V);
    s += fmt("      for (int o = 0; o < %d; ++o) off[o] = 0;\n", nops);
    s += fmt("      for (int d = L.rank - 1; d >= 0; --d) {\n"
             "        %s sh = (%s)L.shape[d]; %s q = lin / sh; %s c = lin - q * sh; lin = q;\n"
             "        for (int o = 0; o < %d; ++o) off[o] += (i64)c * L.st[o][d];\n"
             "      }\n    }\n", IT, IT, IT, IT, nops);
  }
  // input feeds (all loads first, as in the interpreter)
  for (int k = 0; k < P.n_in; ++k) {
    if (RS && RS[k] >= 0) continue;  // a row sum of another input (below)
    const int md = (int)((modes >> (2 * (k + 1))) & 3);
    const bool bl = P.in_dtype[k] == PFB_BOOL;
    const char* T = bl ? "unsigned char" : "float";
    s += fmt("    const %s* p%d = reinterpret_cast<const %s*>(ins.p[%d]) + off[%d];\n", T, k, T, k, k + 1);
    const int np = bl ? 1 : nparts(k);
    if (np > 1) {
      // split-K partials: every part loaded first, then summed in split order
      const char* f[4] = {"x", "y", "z", "w"};
      if (V == 4 && md == 0) {
        for (int q = 0; q < np; ++q)
          s += fmt("    const float4 w%d_%d = __ldg(reinterpret_cast<const float4*>(p%d + %d * PT.st[%d]));\n",
                   k, q, k, q, k);
        for (int j = 0; j < 4; ++j) {
          std::string e = fmt("w%d_0.%s", k, f[j]);
          for (int q = 1; q < np; ++q) e = "(" + e + fmt(" + w%d_%d.%s)", k, q, f[j]);
          s += fmt("    const float in%d_%d = ", k, j) + e + ";\n";
        }
      } else {
        if (md != 1) s += fmt("    const i64 sin%d = L.st[%d][ir];\n", k, k + 1);
        const int nv = md == 1 ? 1 : V;
        for (int j = 0; j < nv; ++j) {
          for (int q = 0; q < np; ++q)
            s += fmt("    const float r%d_%d_%d = __ldg(p%d + %d * PT.st[%d]%s);\n", k, j, q, k, q, k,
                     md == 1 ? "" : fmt(" + %d * sin%d", j, k).c_str());
          std::string e = fmt("r%d_%d_0", k, j);
          for (int q = 1; q < np; ++q) e = "(" + e + fmt(" + r%d_%d_%d)", k, j, q);
          s += fmt("    const float in%d_%d = ", k, j) + e + ";\n";
        }
        for (int j = nv; j < V; ++j) s += fmt("    const float in%d_%d = in%d_0;\n", k, j, k);
      }
    } else if (V == 4 && md == 0) {
      if (bl)
        s += fmt("    const uchar4 w%d = __ldg(reinterpret_cast<const uchar4*>(p%d));\n", k, k);
      else
        s += fmt("    const float4 w%d = __ldg(reinterpret_cast<const float4*>(p%d));\n", k, k);
      const char* f[4] = {"x", "y", "z", "w"};
      for (int j = 0; j < 4; ++j) s += fmt("    const float in%d_%d = (float)w%d.%s;\n", k, j, k, f[j]);
    } else if (md == 1) {
      s += fmt("    const float in%d_0 = (float)__ldg(p%d);\n", k, k);
      for (int j = 1; j < V; ++j) s += fmt("    const float in%d_%d = in%d_0;\n", k, j, k);
    } else {
      s += fmt("    const i64 sin%d = L.st[%d][ir];\n", k, k + 1);
      for (int j = 0; j < V; ++j)
        s += fmt("    const float in%d_%d = (float)__ldg(p%d + %d * sin%d);\n", k, j, k, j, k);
    }
  }
  // row-sum feeds (pass F16): input k = the sum of input RS[k] over the row
  // (the layout's innermost dim, one row per block of blockDim = W threads,
  // V = 1): each thread's value, a fixed xor-shuffle tree per warp, then the
  // warps' sums left to right -- the same order in every block
  if (RS) {
    bool any = false;
    for (int k = 0; k < P.n_in; ++k) {
      if (RS[k] < 0) continue;
      const std::string x = unary_expr(RS[k] >> 16, fmt("in%d_0", RS[k] & 0xffff));
      if (lpr > 0) {  // short rows: a segmented xor tree inside each lpr-lane group
        s += fmt("    float in%d_0;\n    { float v = valid ? ", k) + x + " : 0.f;\n";
        s += fmt("      for (int o = %d; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);\n",
                 lpr / 2);
        s += fmt("      in%d_0 = v; }\n", k);
        continue;
      }
      if (!any) s += "    __shared__ float rs_red[32];\n    const int rs_w = threadIdx.x >> 5, rs_l = threadIdx.x & 31;\n";
      any = true;
      s += fmt("    float in%d_0;\n    { float v = ", k) + x + ";\n";
      s += "      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);\n"
           "      if (rs_l == 0) rs_red[rs_w] = v;\n      __syncthreads();\n"
           "      float t = rs_red[0];\n      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t += rs_red[w];\n"
           "      __syncthreads();\n";
      s += fmt("      in%d_0 = t; }\n", k);
    }
  }
  // the program: reg -> current SSA name
  std::string reg[kMaxRegs];
  for (int r = 0; r < kMaxRegs; ++r) reg[r] = "";
  auto R = [&](int r, int j) { return reg[r].empty() ? std::string("0.f") : reg[r] + "_" + std::to_string(j); };
  for (int st = 0; st < P.n_steps; ++st) {
    const int op = P.code[st][0], dst = P.code[st][1], z = P.code[st][2], w = P.code[st][3];
    const std::string nm = "v" + std::to_string(st);
    for (int j = 0; j < V; ++j) {
      std::string e;
      if (op == F_LOAD) {
        e = z < P.n_in ? fmt("in%d_%d", z, j) : std::string("0.f");
      } else if (op == F_CONST) {
        e = fmt("__int_as_float(%d)", z);
      } else if (op == F_SELECT) {
        e = "(" + R(z, j) + " != 0.f ? " + R(w, j) + " : " + R(dst, j) + ")";
      } else {
        const std::string x = R(z, j), y = R(w, j);
        switch (op) {
          case PFB_ADD: e = x + " + " + y; break;
          case PFB_SUB: e = x + " - " + y; break;
          case PFB_MUL: e = x + " * " + y; break;
          case PFB_DIV: e = x + " / " + y; break;
          case PFB_MAX: e = "np_max(" + x + ", " + y + ")"; break;
          case PFB_MIN: e = "np_min(" + x + ", " + y + ")"; break;
          case PFB_LESS: e = "(" + x + " < " + y + " ? 1.f : 0.f)"; break;
          case PFB_EQUAL: e = "(" + x + " == " + y + " ? 1.f : 0.f)"; break;
          case 16 + PFB_NEG: e = "-" + x; break;
          case 16 + PFB_EXP: e = "expf(" + x + ")"; break;
          case 16 + PFB_LOG: e = "logf(" + x + ")"; break;
          case 16 + PFB_RELU: e = "np_max(" + x + ", 0.f)"; break;
          case 16 + PFB_TANH: e = "tanhf(" + x + ")"; break;
          case 16 + PFB_SIGMOID: e = "1.f / (1.f + expf(-" + x + "))"; break;
          case 16 + PFB_SQUARE: e = x + " * " + x; break;
          case 16 + PFB_LOGICAL_NOT: e = "(" + x + " == 0.f ? 1.f : 0.f)"; break;
          case 66: e = "(" + x + " != 0.f ? 1.f : 0.f)"; break;
          default: e = x; break;  // 67: move
        }
      }
      s += fmt("    const float %s_%d = ", nm.c_str(), j) + e + ";\n";
    }
    reg[dst] = nm;
  }
  // outputs at operand 0's offsets
  const bool vec = (modes & 3) == 0;
  s += "    const i64 so = L.st[0][ir];\n    (void)so;\n";
  if (lpr > 0) s += "    if (!valid) continue;\n";
  for (int k = 0; k < P.n_out; ++k) {
    const int r = P.out_reg[k];
    if (P.out_dt[k] == PFB_BOOL) {
      s += fmt("    { unsigned char* q = reinterpret_cast<unsigned char*>(outs.p[%d]) + off[0];\n", k);
      if (V == 4 && vec)
        s += "      *reinterpret_cast<uchar4*>(q) = make_uchar4(" + R(r, 0) + " != 0.f, " + R(r, 1) +
             " != 0.f, " + R(r, 2) + " != 0.f, " + R(r, 3) + " != 0.f); }\n";
      else {
        for (int j = 0; j < V; ++j) s += fmt("      q[%d * so] = (unsigned char)(", j) + R(r, j) + " != 0.f);\n";
        s += "    }\n";
      }
    } else {
      s += fmt("    { float* q = reinterpret_cast<float*>(outs.p[%d]) + off[0];\n", k);
      if (V == 4 && vec)
        s += "      *reinterpret_cast<float4*>(q) = make_float4(" + R(r, 0) + ", " + R(r, 1) + ", " +
             R(r, 2) + ", " + R(r, 3) + "); }\n";
      else {
        for (int j = 0; j < V; ++j) s += fmt("      q[%d * so] = ", j) + R(r, j) + ";\n";
        s += "    }\n";
      }
    }
  }
  s += "  }\n}\n";
  return s;
}

// integer domain (elementwise.cu fused_int_kernel): i64 registers, numpy
// int64 wraparound through uint64 arithmetic, bool = 0/1, one element per
// thread; ops the integer interpreter does not define move their operand
std::string gen_source_int(const FusedProgram& P, bool idx64) {
  std::string s = fmt(kPrelude, kMaxRank, kMaxFOps, kMaxRank, kMaxOuts, kMaxIn);
  s += "typedef unsigned long long u64;\n";
  const char* IT = idx64 ? "i64" : "unsigned";
  const int nops = P.n_in + 1;
  s += fmt("extern \"C\" __global__ void __launch_bounds__(256) pfb_fused_jit(Layout L, %s n, "
           "Outs outs, Ins ins) {\n", IT);
  s += "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n"
       "  asm volatile(\"griddepcontrol.launch_dependents;\" :::);\n";
  s += fmt("  for (%s e = blockIdx.x * (%s)blockDim.x + threadIdx.x; e < n; "
           "e += (%s)gridDim.x * blockDim.x) {\n", IT, IT, IT);
  s += fmt("    i64 off[%d];\n", nops);
  s += fmt("    if (L.rank == 1) { for (int o = 0; o < %d; ++o) off[o] = (i64)e * L.st[o][0]; }\n", nops);
  s += fmt("    else { %s lin = e;\n", IT);
  s += fmt("      for (int o = 0; o < %d; ++o) off[o] = 0;\n", nops);
  s += fmt("      for (int d = L.rank - 1; d >= 0; --d) {\n"
           "        %s sh = (%s)L.shape[d]; %s q = lin / sh; %s c = lin - q * sh; lin = q;\n"
           "        for (int o = 0; o < %d; ++o) off[o] += (i64)c * L.st[o][d];\n"
           "      }\n    }\n", IT, IT, IT, IT, nops);
  for (int k = 0; k < P.n_in; ++k) {
    if (P.in_dtype[k] == PFB_BOOL)
      s += fmt("    const i64 in%d = (i64)__ldg(reinterpret_cast<const unsigned char*>(ins.p[%d]) + off[%d]);\n",
               k, k, k + 1);
    else
      s += fmt("    const i64 in%d = __ldg(reinterpret_cast<const long long*>(ins.p[%d]) + off[%d]);\n",
               k, k, k + 1);
  }
  std::string reg[kMaxRegs];
  auto R = [&](int r) { return reg[r].empty() ? std::string("(i64)0") : reg[r]; };
  for (int st = 0; st < P.n_steps; ++st) {
    const int op = P.code[st][0], dst = P.code[st][1], z = P.code[st][2], w = P.code[st][3];
    std::string e;
    if (op == F_LOAD) {
      e = z < P.n_in ? fmt("in%d", z) : std::string("(i64)0");
    } else if (op == F_CONST) {
      e = fmt("(i64)(%d)", z);
    } else if (op == F_SELECT) {
      e = "(" + R(z) + " != 0 ? " + R(w) + " : " + R(dst) + ")";
    } else {
      const std::string a = R(z), b = R(w);
      const std::string ua = "(u64)" + a, ub = "(u64)" + b;
      switch (op) {
        case PFB_ADD: e = "(i64)(" + ua + " + " + ub + ")"; break;
        case PFB_SUB: e = "(i64)(" + ua + " - " + ub + ")"; break;
        case PFB_MUL: e = "(i64)(" + ua + " * " + ub + ")"; break;
        case PFB_MAX: e = "(" + a + " >= " + b + " ? " + a + " : " + b + ")"; break;
        case PFB_MIN: e = "(" + a + " <= " + b + " ? " + a + " : " + b + ")"; break;
        case PFB_LESS: e = "(i64)(" + a + " < " + b + ")"; break;
        case PFB_EQUAL: e = "(i64)(" + a + " == " + b + ")"; break;
        case 16 + PFB_NEG: e = "(i64)((u64)0 - " + ua + ")"; break;
        case 16 + PFB_SQUARE: e = "(i64)(" + ua + " * " + ua + ")"; break;
        case 16 + PFB_LOGICAL_NOT: e = "(i64)(" + a + " == 0)"; break;
        case 66: e = "(i64)(" + a + " != 0)"; break;
        default: e = a; break;
      }
    }
    const std::string nm = "v" + std::to_string(st);
    s += "    const i64 " + nm + " = " + e + ";\n";
    reg[dst] = nm;
  }
  for (int k = 0; k < P.n_out; ++k) {
    if (P.out_dt[k] == PFB_BOOL)
      s += fmt("    reinterpret_cast<unsigned char*>(outs.p[%d])[off[0]] = (unsigned char)(", k) +
           R(P.out_reg[k]) + " != 0);\n";
    else if (P.out_dt[k] == PFB_F32)
      s += fmt("    reinterpret_cast<float*>(outs.p[%d])[off[0]] = (float)", k) + R(P.out_reg[k]) + ";\n";
    else
      s += fmt("    reinterpret_cast<long long*>(outs.p[%d])[off[0]] = ", k) + R(P.out_reg[k]) + ";\n";
  }
  s += "  }\n}\n";
  return s;
}

// NVRTC: source -> sm_100a cubin (empty on failure; the log goes to stderr)
std::string to_cubin(const std::string& src) {
  const Nvrtc& N = nvrtc();
  nvrtcProgram prog;
  if (N.create(&prog, src.c_str(), "pfb_fused_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return {};
  const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17",
                        "-default-device", "-lineinfo"};
  nvrtcResult rc = N.compile(prog, 5, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    N.log_size(prog, &n);
    std::string log(n, '\0');
    N.log(prog, &log[0]);
    fprintf(stderr, "pfb: fused-program compile failed (interpreter used):\n%s\n", log.c_str());
    N.destroy(&prog);
    return {};
  }
  size_t n = 0;
  N.cubin_size(prog, &n);
  std::string cubin(n, '\0');
  N.cubin(prog, &cubin[0]);
  N.destroy(&prog);
  return cubin;
}

CUfunction compile(const std::string& src) {
  const std::string cubin = to_cubin(src);
  if (cubin.empty()) return nullptr;
  const Driver& D = driver();
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  // a load is not a stream operation; allow it while this thread captures
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  CUresult r = D.load(&mod, cubin.data());
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (r != CUDA_SUCCESS || D.get(&fn, mod, "pfb_fused_jit") != CUDA_SUCCESS) return nullptr;
  return fn;
}

int g_jit_on = -1;           // -1: not yet read from PFB_NO_JIT
int64_t g_jit_min = 0;       // PFB_JIT_MIN: smallest group specialised
int64_t g_jit_layout_min = 32768;  // PFB_JIT_LAYOUT_MIN: smallest group with its layout baked in

void jit_init() {
  if (g_jit_on >= 0) return;
  g_jit_on = getenv_flag("PFB_NO_JIT") ? 0 : 1;
  if (const char* e = getenv("PFB_JIT_MIN")) g_jit_min = atoll(e);
  if (const char* e = getenv("PFB_JIT_LAYOUT_MIN")) g_jit_layout_min = atoll(e);
}

}  // namespace

namespace {

// kernel for a program (integer: the i64 domain), compiled on first use
CUfunction lookup(const FusedProgram& P, int V, bool idx64, FeedModes modes, bool integer,
                  const PartsSpec* PS = nullptr, const FLayout* LS = nullptr, bool off32 = false,
                  const int* RS = nullptr, int lpr = 0) {
  int dev = 0;
  cudaGetDevice(&dev);
  // cache key: the program's encoding and everything baked into the source
  int32_t kb[16 + 3 * kMaxIn + 4 * kMaxSteps + 2 * kMaxOuts + 2 * kMaxRank * (kMaxFOps + 1)];
  int nk = 0;
  kb[nk++] = dev; kb[nk++] = V; kb[nk++] = idx64; kb[nk++] = (int32_t)(modes & 0xffffffffu);
  kb[nk++] = (int32_t)(modes >> 32); kb[nk++] = integer;
  kb[nk++] = P.n_in; kb[nk++] = P.n_steps; kb[nk++] = P.n_out;
  for (int k = 0; k < P.n_in; ++k) kb[nk++] = P.in_dtype[k];
  for (int t = 0; t < P.n_steps; ++t)
    for (int j = 0; j < 4; ++j) kb[nk++] = P.code[t][j];
  for (int k = 0; k < P.n_out; ++k) { kb[nk++] = P.out_reg[k]; kb[nk++] = P.out_dt[k]; }
  kb[nk++] = PS != nullptr;
  if (PS)
    for (int k = 0; k < P.n_in; ++k) kb[nk++] = PS->S[k];
  kb[nk++] = RS != nullptr;
  kb[nk++] = lpr;
  if (RS)
    for (int k = 0; k < P.n_in; ++k) kb[nk++] = RS[k];
  kb[nk++] = LS != nullptr;
  if (LS) {  // the layout baked into the source (64-bit values as two words)
    kb[nk++] = LS->rank;
    kb[nk++] = off32;
    for (int d = 0; d < LS->rank; ++d) {
      kb[nk++] = (int32_t)LS->shape[d];
      kb[nk++] = (int32_t)(LS->shape[d] >> 32);
      for (int o = 0; o <= P.n_in; ++o) {
        kb[nk++] = (int32_t)LS->st[o][d];
        kb[nk++] = (int32_t)(LS->st[o][d] >> 32);
      }
    }
  }
  const std::string key(reinterpret_cast<const char*>(kb), nk * sizeof(int32_t));
  static std::mutex mu;
  static std::unordered_map<std::string, CUfunction> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it == cache.end())
    it = cache.emplace(key, compile(integer ? gen_source_int(P, idx64)
                                            : gen_source(P, V, idx64, modes, PS, LS, off32, RS, lpr))).first;
  return it->second;
}

bool run(CUfunction fn, bool idx64, const FLayout& L, int64_t nitems, const FusedOuts& outs,
         const FusedIns& ins, cudaStream_t s, const PartsSpec* PS = nullptr, int block = 256) {
  CUlaunchConfig cfg = {};
  cfg.gridDimX = grid_for(nitems, block); cfg.gridDimY = 1; cfg.gridDimZ = 1;
  cfg.blockDimX = block; cfg.blockDimY = 1; cfg.blockDimZ = 1;
  cfg.hStream = (CUstream)s;
  CUlaunchAttribute attr[1];
  attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  attr[0].value.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  FLayout Lc = L;
  FusedOuts oc = outs;
  FusedIns ic = ins;
  uint32_t n32 = (uint32_t)nitems;
  int64_t n64 = nitems;
  struct { int64_t st[kMaxIn]; } pt;
  if (PS)
    for (int k = 0; k < kMaxIn; ++k) pt.st[k] = PS->st[k];
  void* args[5] = {&Lc, idx64 ? (void*)&n64 : (void*)&n32, &oc, &ic, &pt};
  kernel_launches()++;
  return driver().launch(&cfg, fn, args, nullptr) == CUDA_SUCCESS;
}

bool usable(int64_t elems) {
  jit_init();
  return g_jit_on && elems >= g_jit_min && nvrtc().ok && driver().ok;
}

}  // namespace

bool fused_jit_launch(const FusedProgram& P, int V, bool idx64, FeedModes modes, const FLayout& L,
                      int64_t ngroups, const FusedOuts& outs, const FusedIns& ins,
                      cudaStream_t s, const PartsSpec* parts) {
  if (parts && !parts->any()) parts = nullptr;
  if (!usable(parts ? INT64_MAX : ngroups * V)) return false;
  // groups of >= 32K elements (the ones a step repeats: cfg4's cell, cfg5's
  // select) get the layout baked in; small ones share one kernel per program
  const FLayout* LS = ngroups * V >= g_jit_layout_min ? &L : nullptr;
  bool off32 = false;
  if (LS) {
    double mx = 0;
    for (int o = 0; o <= P.n_in; ++o) {
      double m = 0;
      for (int d = 0; d < L.rank; ++d) m += (double)(L.shape[d] - 1) * std::fabs((double)L.st[o][d]);
      mx = std::max(mx, m);
    }
    off32 = mx < 2147483647.0;
  }
  CUfunction fn = lookup(P, V, idx64, modes, false, parts, LS, off32);
  return fn && run(fn, idx64, L, ngroups, outs, ins, s, parts);
}

bool fused_rows_jit_launch(const FusedProgram& P, FeedModes modes, const FLayout& L,
                           int64_t n, const FusedOuts& outs, const FusedIns& ins, cudaStream_t s,
                           const PartsSpec* parts, const int* rowsum) {
  if (parts && !parts->any()) parts = nullptr;
  if (!usable(INT64_MAX) || L.rank < 1) return false;
  const int ir = L.rank - 1;
  const int64_t W = L.shape[ir];
  // one row per block: W threads, a whole number of warps, rows = every
  // coordinate of the outer dims; each row-sum input broadcasts along the
  // row and varies along every outer dim (so a row is exactly its extent-1
  // axes)
  // rows shorter than a warp: lpr = the next power of two >= W lanes per
  // row, several rows per warp (cfg2's softmax over 10 logits)
  int lpr = 0;
  if (W < 32) {
    lpr = 1;
    while (lpr < W) lpr *= 2;
  } else if (W > 1024 || W % 32 != 0) {
    return false;
  }
  if (n % W != 0) return false;
  for (int k = 0; k < P.n_in; ++k) {
    if (rowsum[k] < 0) continue;
    const int j = rowsum[k] & 0xffff;
    if (j >= P.n_in || j == k || rowsum[j] >= 0 || P.in_dtype[j] != PFB_F32 ||
        L.st[k + 1][ir] != 0)
      return false;
    for (int d = 0; d < ir; ++d)
      if (L.shape[d] > 1 && L.st[k + 1][d] == 0) return false;
  }
  double mx = 0;
  for (int o = 0; o <= P.n_in; ++o) {
    double m = 0;
    for (int d = 0; d < L.rank; ++d) m += (double)(L.shape[d] - 1) * std::fabs((double)L.st[o][d]);
    mx = std::max(mx, m);
  }
  const bool idx64 = n >= (int64_t)0x7fffffff;
  if (lpr > 0) {  // one thread per (row, lane) of the padded rows, whole warps
    const int64_t rows = n / W;
    const int64_t ng = (rows * lpr + 31) / 32 * 32;
    CUfunction fn = lookup(P, 1, idx64 || ng >= (int64_t)0x7fffffff, modes, false, parts, &L,
                           mx < 2147483647.0, rowsum, lpr);
    return fn && run(fn, idx64 || ng >= (int64_t)0x7fffffff, L, ng, outs, ins, s, parts, 256);
  }
  CUfunction fn = lookup(P, 1, idx64, modes, false, parts, &L, mx < 2147483647.0, rowsum);
  return fn && run(fn, idx64, L, n, outs, ins, s, parts, (int)W);
}

bool fused_int_jit_launch(const FusedProgram& P, bool idx64, const FLayout& L, int64_t n,
                          const FusedOuts& outs, const FusedIns& ins, cudaStream_t s) {
  if (!usable(n)) return false;
  CUfunction fn = lookup(P, 1, idx64, 0, true);
  return fn && run(fn, idx64, L, n, outs, ins, s);
}

}  // namespace pfb

// Runtime control of the specialiser (tests compare it with the interpreter):
// enable 0/1, min_elems < 0 keeps the current threshold.  Returns 1 when the
// specialiser can run on this process (NVRTC + driver entry points found).
extern "C" int pfb_fused_jit_config(int32_t enable, int64_t min_elems) {
  pfb::jit_init();
  pfb::g_jit_on = enable ? 1 : 0;
  if (min_elems >= 0) pfb::g_jit_min = min_elems;
  return pfb::nvrtc().ok && pfb::driver().ok;
}

// Can fused groups take split-K partial-sum inputs (pfb_fused_ew_parts) in
// this process right now (specialiser available and enabled)?
extern "C" int pfb_fused_parts_ok(void) { return pfb::usable(INT64_MAX) ? 1 : 0; }

// Host-only check (no device needed): generate the specialised source for a
// program and compile it with NVRTC for sm_100a.  0 = compiled, 1 = compile
// error (log on stderr), PFB_E_UNSUPPORTED = NVRTC not found, PFB_E_ARG = bad
// program.  integer != 0 selects the i64/bool domain (v ignored).
extern "C" int pfb_fused_jit_check(int32_t integer, int32_t v, uint64_t modes, int32_t n_in,
                                   const int32_t* in_dtypes, int32_t n_steps,
                                   const int32_t* program, int32_t n_out, const int32_t* out_regs,
                                   const int32_t* out_dtypes) {
  using namespace pfb;
  if (n_in < 1 || n_in > kMaxIn || n_steps < 1 || n_steps > kMaxSteps || n_out < 1 ||
      n_out > kMaxOuts || (v != 1 && v != 4))
    return PFB_E_ARG;
  if (!nvrtc().ok) return PFB_E_UNSUPPORTED;
  FusedProgram P{};
  P.n_in = n_in;
  P.n_steps = n_steps;
  P.n_out = n_out;
  for (int k = 0; k < n_in; ++k) P.in_dtype[k] = in_dtypes[k];
  for (int t = 0; t < n_steps; ++t) {
    for (int j = 0; j < 4; ++j) P.code[t][j] = program[4 * t + j];
    if (P.code[t][1] < 0 || P.code[t][1] >= kMaxRegs) return PFB_E_ARG;
  }
  for (int k = 0; k < n_out; ++k) {
    if (out_regs[k] < 0 || out_regs[k] >= kMaxRegs) return PFB_E_ARG;
    P.out_reg[k] = out_regs[k];
    P.out_dt[k] = out_dtypes[k];
  }
  const std::string src = integer ? gen_source_int(P, false) : gen_source(P, v, false, modes);
  return to_cubin(src).empty() ? 1 : 0;
}
