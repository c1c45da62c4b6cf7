// pfb_matmul: validation + path selection (reference tensor.py:195-206).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "gemm.cuh"

using namespace pfb;

static int matmul_args(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out, GemmArgs* g) {
  if (a->dtype != b->dtype) return PFB_E_DTYPE;
  if (a->dtype != PFB_F32 || out->dtype != PFB_F32) return PFB_E_DTYPE;  // int matmul: not on the path
  if (a->rank == 2 && b->rank == 2) {
    if (a->shape[1] != b->shape[0]) return PFB_E_SHAPE;
    if (out->rank != 2 || out->shape[0] != a->shape[0] || out->shape[1] != b->shape[1])
      return PFB_E_SHAPE;
    *g = GemmArgs{1, a->shape[0], b->shape[1], a->shape[1],
                  (const float*)a->data, 0, a->stride[0], a->stride[1],
                  (const float*)b->data, 0, b->stride[0], b->stride[1],
                  (float*)out->data, 0, out->stride[0], out->stride[1], nullptr, 0};
    return 0;
  }
  if (a->rank == 3 && b->rank == 3) {
    if (a->shape[0] != b->shape[0] || a->shape[2] != b->shape[1]) return PFB_E_SHAPE;
    if (out->rank != 3 || out->shape[0] != a->shape[0] || out->shape[1] != a->shape[1] ||
        out->shape[2] != b->shape[2])
      return PFB_E_SHAPE;
    *g = GemmArgs{a->shape[0], a->shape[1], b->shape[2], a->shape[2],
                  (const float*)a->data, a->stride[0], a->stride[1], a->stride[2],
                  (const float*)b->data, b->stride[0], b->stride[1], b->stride[2],
                  (float*)out->data, out->stride[0], out->stride[1], out->stride[2], nullptr, 0};
    return 0;
  }
  return PFB_E_RANK;
}

__global__ void zero_f32(float* p, int64_t n) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.f;
}

// Per-shape autotuning of the tcgen05-vs-SIMT choice: on the first call of a
// shape (outside stream capture, not accumulating) both paths run twice and
// the faster second run wins; later calls -- including the ones captured into
// CUDA graphs -- reuse the cached choice.  PFB_GEMM_AUTOTUNE=0 uses the model.
namespace {
using ShapeKey = std::tuple<int64_t, int64_t, int64_t, int64_t, int, int, int, int, int>;
std::map<ShapeKey, int> g_choice;  // 1 = SIMT, 3 = tcgen05 pre-split, 4 = tcgen05 raw feed
std::mutex g_mu;

ShapeKey key_of(const GemmArgs& g) {
  return ShapeKey(g.batch, g.M, g.N, g.K, g.sak == 1, g.sam == 1, g.sbk == 1, g.sbn == 1,
                  (g.sab == 0 ? 1 : (g.sbb == 0 ? 2 : 0)) + 4 * gemm_tcgen05_raw_possible(g) +
                      8 * (g.b_hi != nullptr));
}

// PFB_GEMM_TUNE_FILE: persist choices across processes (a profiling run under
// ncu replays the choices of an unprofiled run instead of re-timing under the
// profiler).  One line per shape: the 9 key fields and the path.
const char* tune_file() {
  static const char* f = getenv("PFB_GEMM_TUNE_FILE");
  return (f && f[0]) ? f : nullptr;
}

void load_tune_file() {
  static bool done = false;
  if (done) return;
  done = true;
  const char* fn = tune_file();
  if (!fn) return;
  FILE* f = fopen(fn, "r");
  if (!f) return;
  long long v[10];
  while (fscanf(f, "%lld %lld %lld %lld %lld %lld %lld %lld %lld %lld", &v[0], &v[1], &v[2],
                &v[3], &v[4], &v[5], &v[6], &v[7], &v[8], &v[9]) == 10)
    g_choice[ShapeKey(v[0], v[1], v[2], v[3], (int)v[4], (int)v[5], (int)v[6], (int)v[7],
                      (int)v[8])] = (int)v[9];
  fclose(f);
}

void save_choice(const ShapeKey& k, int path) {
  const char* fn = tune_file();
  if (!fn) return;
  FILE* f = fopen(fn, "a");
  if (!f) return;
  fprintf(f, "%lld %lld %lld %lld %d %d %d %d %d %d\n", (long long)std::get<0>(k),
          (long long)std::get<1>(k), (long long)std::get<2>(k), (long long)std::get<3>(k),
          std::get<4>(k), std::get<5>(k), std::get<6>(k), std::get<7>(k), std::get<8>(k), path);
  fclose(f);
}

bool tc_pair_off() {
  static const bool off = getenv_flag("PFB_DISABLE_PAIR");
  return off;
}

bool autotune_enabled() {
  static const bool on = [] {
    const char* e = getenv("PFB_GEMM_AUTOTUNE");
    return !(e && e[0] == '0');
  }();
  return on;
}

int run_path(const GemmArgs& g, int path, void* ws, int64_t ws_bytes, cudaStream_t s) {
  switch (path) {
    case 1: return gemm_simt(g, ws, ws_bytes, s);
    case 10: return gemm_simt_v(g, ws, ws_bytes, s, 4, false);  // SIMT, 4 k-splits (cluster)
    case 11: return gemm_simt_v(g, ws, ws_bytes, s, 16, true);  // SIMT, 16 k-splits (workspace)
    case 3: return gemm_tcgen05(g, ws, ws_bytes, s, 1);
    case 4: return gemm_tcgen05(g, ws, ws_bytes, s, 2);
    case 7: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 2);  // raw feed, 2 / 4 k-splits
    case 8: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 4);
    case 9: return gemm_tcgen05(g, ws, ws_bytes, s, 1, 4);  // pre-split, 4 k-splits
    // narrow tiles (skinny M: N-parallel instead of k-split reductions)
    case 12: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 0, 64);
    case 13: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 0, 32);
    case 14: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 2, 32);
    case 15: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 4, 32);
    case 16: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 2, 64);
    case 17: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 4, 64);
    case 18: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 8, 64);
    case 19: return gemm_tcgen05(g, ws, ws_bytes, s, 2, 8, 32);
    case 5: return gemm_tcgen05_pair(g, ws, ws_bytes, s, 1);
    case 6: return gemm_tcgen05_pair(g, ws, ws_bytes, s, 2);
    default: return gemm_tcgen05(g, ws, ws_bytes, s, 0);
  }
}

float time_path(const GemmArgs& g, int path, void* ws, int64_t ws_bytes, cudaStream_t s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 1e30f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0, s);
    int rc = run_path(g, path, ws, ws_bytes, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    if (rc != 0) { ms = 1e30f; break; }
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}
}  // namespace

extern "C" int64_t pfb_matmul_workspace(const pfb_tensor* a, const pfb_tensor* b,
                                        pfb_tensor* out) {
  GemmArgs g;
  if (matmul_args(a, b, out, &g)) return 0;
  return std::max(std::max(gemm_tcgen05_workspace(g), gemm_simt_workspace(g)),
                  gemm_simt_workspace_max(g));
}

static int matmul_impl(GemmArgs& g, pfb_tensor* out, int32_t force_path, void* ws,
                       int64_t ws_bytes, void* stream);

extern "C" int pfb_matmul_ex(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                             const float* alpha_rows, int32_t accumulate, int32_t force_path,
                             void* ws, int64_t ws_bytes, void* stream) {
  return pfb_matmul_fused(a, b, out, nullptr, nullptr, PFB_ACT_NONE, alpha_rows, accumulate,
                          force_path, ws, ws_bytes, stream);
}

extern "C" int pfb_matmul_fused(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                                const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                                const float* alpha_rows, int32_t accumulate, int32_t force_path,
                                void* ws, int64_t ws_bytes, void* stream) {
  return pfb_matmul_ep(a, b, out, kscale, bias, act, nullptr, PFB_DOP_NONE, alpha_rows, accumulate,
                       force_path, ws, ws_bytes, stream);
}

static int matmul_ep_impl(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                          const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                          const pfb_tensor* dy, int32_t dop, const float* alpha_rows,
                          int32_t accumulate, const void* b_planes, int32_t force_path, void* ws,
                          int64_t ws_bytes, void* stream);

extern "C" int pfb_matmul_ep(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                             const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                             const pfb_tensor* dy, int32_t dop, const float* alpha_rows,
                             int32_t accumulate, int32_t force_path, void* ws, int64_t ws_bytes,
                             void* stream) {
  return matmul_ep_impl(a, b, out, kscale, bias, act, dy, dop, alpha_rows, accumulate, nullptr,
                        force_path, ws, ws_bytes, stream);
}

// B as the GEMM consumes it: batch, K, N and the batch stride of a [K, N] or
// [batch, K, N] view (batch stride 0 = one matrix shared by the batch)
static bool planes_args(const pfb_tensor* b, GemmArgs* g) {
  if (b->dtype != PFB_F32 || (b->rank != 2 && b->rank != 3)) return false;
  const int r = b->rank;
  *g = GemmArgs{r == 3 ? b->shape[0] : 1, 1, b->shape[r - 1], b->shape[r - 2],
                nullptr, 0, 0, 1, (const float*)b->data, r == 3 ? b->stride[0] : 0,
                b->stride[r - 2], b->stride[r - 1], nullptr, 0, 0, 1, nullptr, 0};
  return g->K > 0 && g->N > 0;
}

static const float* planes_lo(const GemmArgs& g, const void* planes) {
  return reinterpret_cast<const float*>(static_cast<const char*>(planes) + gemm_planes_bytes(g) / 2);
}

extern "C" int64_t pfb_gemm_planes_bytes(const pfb_tensor* b) {
  GemmArgs g;
  return planes_args(b, &g) ? gemm_planes_bytes(g) : 0;
}

extern "C" int pfb_gemm_split_planes(const pfb_tensor* b, void* planes, void* stream) {
  GemmArgs g;
  if (!planes_args(b, &g) || planes == nullptr) return PFB_E_ARG;
  const int64_t Kp = (g.K + 3) / 4 * 4;
  const int64_t bb = (g.sbb == 0 && g.batch > 1) ? 1 : g.batch;
  float* hi = static_cast<float*>(planes);
  tc_split_launch(g.B, bb, g.N, g.K, Kp, g.sbb, g.sbn, g.sbk, hi, const_cast<float*>(planes_lo(g, planes)),
                  nullptr, 0, 0, as_stream(stream));
  return launch_status();
}

extern "C" int pfb_matmul_ep2(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                              const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                              const pfb_tensor* dy, int32_t dop, const void* b_planes,
                              int32_t force_path, void* ws, int64_t ws_bytes, void* stream) {
  return matmul_ep_impl(a, b, out, kscale, bias, act, dy, dop, nullptr, 0, b_planes, force_path,
                        ws, ws_bytes, stream);
}

static int matmul_ep_impl(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out,
                          const pfb_tensor* kscale, const pfb_tensor* bias, int32_t act,
                          const pfb_tensor* dy, int32_t dop, const float* alpha_rows,
                          int32_t accumulate, const void* b_planes, int32_t force_path, void* ws,
                          int64_t ws_bytes, void* stream) {
  GemmArgs g;
  if (int e = matmul_args(a, b, out, &g)) return e;
  if (b_planes != nullptr && kscale == nullptr) {
    g.b_hi = static_cast<const float*>(b_planes);
    g.b_lo = planes_lo(g, b_planes);
  }
  g.alpha_rows = alpha_rows;
  g.accumulate = accumulate;
  if (act < PFB_ACT_NONE || act > PFB_ACT_RELU) return PFB_E_ARG;
  g.act = act;
  const bool batched = a->rank == 3;
  if (bias) {
    if (bias->dtype != PFB_F32) return PFB_E_DTYPE;
    int64_t st[3];
    if (!broadcast_strides(bias, out->rank, out->shape, st)) return PFB_E_SHAPE;
    g.bias = (const float*)bias->data;
    if (batched) { g.sxb = st[0]; g.sxm = st[1]; g.sxn = st[2]; }
    else { g.sxb = 0; g.sxm = st[0]; g.sxn = st[1]; }
  }
  if (kscale) {
    if (kscale->dtype != PFB_F32) return PFB_E_DTYPE;
    const int64_t shp[2] = {g.batch, g.K};
    int64_t st[2];
    if (batched) {
      if (!broadcast_strides(kscale, 2, shp, st)) return PFB_E_SHAPE;
      g.skb = st[0]; g.skk = st[1];
    } else {
      if (!broadcast_strides(kscale, 1, shp + 1, st)) return PFB_E_SHAPE;
      g.skb = 0; g.skk = st[0];
    }
    g.kscale = (const float*)kscale->data;
  }
  if (dop < PFB_DOP_NONE || dop > PFB_DOP_DSIGMOID || (dop && dy == nullptr)) return PFB_E_ARG;
  if (dop) {
    if (dy->dtype != PFB_F32) return PFB_E_DTYPE;
    int64_t st[3];
    if (!broadcast_strides(dy, out->rank, out->shape, st)) return PFB_E_SHAPE;
    g.dy = (const float*)dy->data;
    g.dop = dop;
    if (batched) { g.sdb = st[0]; g.sdm = st[1]; g.sdn = st[2]; }
    else { g.sdb = 0; g.sdm = st[0]; g.sdn = st[1]; }
  }
  if (g.K == 0 && (g.has_epi() || g.kscale)) return PFB_E_UNSUPPORTED;
  return matmul_impl(g, out, force_path, ws, ws_bytes, stream);
}

static int matmul_impl(GemmArgs& g, pfb_tensor* out, int32_t force_path, void* ws,
                       int64_t ws_bytes, void* stream) {
  const int accumulate = g.accumulate;
  cudaStream_t s = as_stream(stream);
  if (g.batch == 0 || g.M == 0 || g.N == 0) return 0;
  if (g.K == 0) {
    if (accumulate) return 0;
    if (!is_dense(out)) return PFB_E_UNSUPPORTED;
    int64_t n = numel(out);
    launch(zero_f32, grid_for(n, 256), 256, 0, s, (float*)out->data, n);
    return launch_status();
  }
  // force_path: 0 = auto, 1 = SIMT, 2 = tcgen05 (error if ineligible),
  // 3 = tcgen05 with pre-split operands, 4 = tcgen05 with the raw TMA feed,
  // 5 / 6 = CTA-pair tcgen05 (cta_group::2) with pre-split / raw operands.
  // PFB_DISABLE_TCGEN05=1 pins auto to SIMT (A/B testing, bring-up).
  static const bool tc_off = getenv("PFB_DISABLE_TCGEN05") && getenv("PFB_DISABLE_TCGEN05")[0] == '1';
  if (force_path >= 1 && force_path <= 19) return run_path(g, force_path, ws, ws_bytes, s);
  const bool tc_ok = !tc_off && gemm_tcgen05_eligible(g) &&
                     ws_bytes >= gemm_tcgen05_workspace(g) && ws != nullptr &&
                     (double)g.batch * g.M * g.N * g.K >= (double)(1 << 20);
  if (!tc_ok) return gemm_simt(g, ws, ws_bytes, s);
  int path = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    load_tune_file();
    auto it = g_choice.find(key_of(g));
    if (it != g_choice.end()) path = it->second;
  }
  if (path == 0) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    if (autotune_enabled() && !accumulate && st == cudaStreamCaptureStatusNone) {
      // every candidate runs twice; the last one timed leaves C computed
      int cand[20];
      int ncand = 0;
      cand[ncand++] = 1;
      if (gemm_simt_splittable(g)) { cand[ncand++] = 10; cand[ncand++] = 11; }
      cand[ncand++] = 3;
      // forced k-splits only where tiles leave SMs idle (the model's split
      // choice is a heuristic; the timing decides)
      const int64_t tiles128 = ((g.M + 127) / 128) * ((g.N + 127) / 128) * g.batch;
      const bool few_tiles = tiles128 < 148 && g.K >= 256;
      if (few_tiles) cand[ncand++] = 9;
      if (gemm_tcgen05_raw_possible(g)) {
        cand[ncand++] = 4;
        if (few_tiles) { cand[ncand++] = 7; cand[ncand++] = 8; }
        if (few_tiles && g.M <= 512)
          for (int c : {12, 13, 14, 15, 16, 17, 18, 19}) cand[ncand++] = c;
      }
      if (g.M > 128 && !tc_pair_off()) {
        cand[ncand++] = 5;
        if (gemm_tcgen05_raw_possible(g)) cand[ncand++] = 6;
      }
      float best = 1e30f;
      for (int i = 0; i < ncand; ++i) {
        const float t = time_path(g, cand[i], ws, ws_bytes, s);
        if (t < best) { best = t; path = cand[i]; }
      }
      {
        std::lock_guard<std::mutex> lk(g_mu);
        g_choice[key_of(g)] = path;
        save_choice(key_of(g), path);
      }
      if (path == cand[ncand - 1]) return launch_status();
      return run_path(g, path, ws, ws_bytes, s);
    }
    path = gemm_tcgen05_profitable(g) ? 2 : 1;
  }
  if (path != 1) {
    int e = run_path(g, path, ws, ws_bytes, s);
    if (e != PFB_E_UNSUPPORTED) return e;
  }
  return gemm_simt(g, ws, ws_bytes, s);
}

extern "C" int pfb_matmul(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* out, void* ws,
                          int64_t ws_bytes, void* stream) {
  return pfb_matmul_ex(a, b, out, nullptr, 0, 0, ws, ws_bytes, stream);
}

// ---------------------------------------------------------------------------
// Two operand pairs into one output (passes.fuse_dual_matmuls):
//   out = act(a1 @ b1 + a2 @ b2 + bias)
// -- matmul(concat([a1, a2], -1), b) with b split at K1, or the sum of two
// matmuls.  The tcgen05 path accumulates both K ranges in one launch; the
// fallback is two GEMM launches, the second accumulating with the epilogue.

namespace {
std::map<std::tuple<ShapeKey, int64_t, int>, int> g_dual_choice;  // 1 two launches, 2 raw, 3 pre-split

int dual_path(const GemmArgs& g1, const GemmArgs& g2, int path, pfb_tensor* out, void* ws,
              int64_t ws_bytes, cudaStream_t s) {
  if (path == 2 || path == 3)
    return gemm_tcgen05_dual(g1, g2, ws, ws_bytes, s, path == 2 ? 2 : 1);
  if (path == 4 || path == 5)  // raw feed, narrow tiles
    return gemm_tcgen05_dual(g1, g2, ws, ws_bytes, s, 2, 0, path == 4 ? 64 : 32);
  GemmArgs h1 = g1, h2 = g2;
  h1.bias = nullptr;
  h1.act = 0;
  h2.accumulate = 1;
  h2.bias = g1.bias;
  h2.sxb = g1.sxb; h2.sxm = g1.sxm; h2.sxn = g1.sxn;
  h2.act = g1.act;
  if (int e = matmul_impl(h1, out, 0, ws, ws_bytes, s)) return e;
  return matmul_impl(h2, out, 0, ws, ws_bytes, s);
}

float time_dual(const GemmArgs& g1, const GemmArgs& g2, int path, pfb_tensor* out, void* ws,
                int64_t ws_bytes, cudaStream_t s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 1e30f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0, s);
    int rc = dual_path(g1, g2, path, out, ws, ws_bytes, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    if (rc != 0) { ms = 1e30f; break; }
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}
}  // namespace

extern "C" int64_t pfb_matmul_dual_workspace(const pfb_tensor* a1, const pfb_tensor* b1,
                                             const pfb_tensor* a2, const pfb_tensor* b2,
                                             pfb_tensor* out) {
  GemmArgs g1, g2;
  if (matmul_args(a1, b1, out, &g1) || matmul_args(a2, b2, out, &g2)) return 0;
  return std::max({gemm_tcgen05_dual_workspace(g1, g2), gemm_tcgen05_workspace(g1),
                   gemm_tcgen05_workspace(g2), gemm_simt_workspace(g1), gemm_simt_workspace(g2)});
}

extern "C" int pfb_matmul_dual(const pfb_tensor* a1, const pfb_tensor* b1, const pfb_tensor* a2,
                               const pfb_tensor* b2, pfb_tensor* out, const pfb_tensor* bias,
                               int32_t act, int32_t force_path, void* ws, int64_t ws_bytes,
                               void* stream) {
  return pfb_matmul_dual2(a1, b1, a2, b2, out, bias, act, nullptr, nullptr, force_path, ws,
                          ws_bytes, stream);
}

extern "C" int pfb_matmul_dual2(const pfb_tensor* a1, const pfb_tensor* b1, const pfb_tensor* a2,
                                const pfb_tensor* b2, pfb_tensor* out, const pfb_tensor* bias,
                                int32_t act, const void* b1_planes, const void* b2_planes,
                                int32_t force_path, void* ws, int64_t ws_bytes, void* stream) {
  GemmArgs g1, g2;
  if (int e = matmul_args(a1, b1, out, &g1)) return e;
  if (int e = matmul_args(a2, b2, out, &g2)) return e;
  if (b1_planes) { g1.b_hi = static_cast<const float*>(b1_planes); g1.b_lo = planes_lo(g1, b1_planes); }
  if (b2_planes) { g2.b_hi = static_cast<const float*>(b2_planes); g2.b_lo = planes_lo(g2, b2_planes); }
  if (act < PFB_ACT_NONE || act > PFB_ACT_RELU) return PFB_E_ARG;
  g1.act = act;
  if (bias) {
    if (bias->dtype != PFB_F32) return PFB_E_DTYPE;
    int64_t st[3];
    if (!broadcast_strides(bias, out->rank, out->shape, st)) return PFB_E_SHAPE;
    g1.bias = (const float*)bias->data;
    if (a1->rank == 3) { g1.sxb = st[0]; g1.sxm = st[1]; g1.sxn = st[2]; }
    else { g1.sxb = 0; g1.sxm = st[0]; g1.sxn = st[1]; }
  }
  cudaStream_t s = as_stream(stream);
  if (g1.batch == 0 || g1.M == 0 || g1.N == 0) return 0;
  static const bool tc_off = getenv_flag("PFB_DISABLE_TCGEN05") || getenv_flag("PFB_DISABLE_DUAL");
  if (force_path >= 1 && force_path <= 5) return dual_path(g1, g2, force_path, out, ws, ws_bytes, s);
  const bool tc_ok = !tc_off && g1.K > 0 && g2.K > 0 && gemm_tcgen05_eligible(g1) &&
                     gemm_tcgen05_eligible(g2) && ws != nullptr &&
                     ws_bytes >= gemm_tcgen05_dual_workspace(g1, g2) &&
                     (double)g1.batch * g1.M * g1.N * (g1.K + g2.K) >= (double)(1 << 20);
  if (!tc_ok) return dual_path(g1, g2, 1, out, ws, ws_bytes, s);
  const auto key = std::make_tuple(key_of(g1), g2.K, (int)(g2.sak == 1) + 2 * (int)(g2.sbk == 1) +
                                                      4 * (int)(g2.b_hi != nullptr));
  int path = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_dual_choice.find(key);
    if (it != g_dual_choice.end()) path = it->second;
  }
  if (path == 0) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    if (!autotune_enabled() || st != cudaStreamCaptureStatusNone)
      return dual_path(g1, g2, 2, out, ws, ws_bytes, s);
    float best = 1e30f;
    const bool skinny = g1.M <= 512 &&
                        ((g1.M + 127) / 128) * ((g1.N + 127) / 128) * g1.batch < 148;
    for (int cand : {1, 3, 2, 4, 5}) {
      if (cand >= 4 && !skinny) continue;
      const float t = time_dual(g1, g2, cand, out, ws, ws_bytes, s);
      if (t < best) { best = t; path = cand; }
    }
    std::lock_guard<std::mutex> lk(g_mu);
    g_dual_choice[key] = path;
  }
  const int e = dual_path(g1, g2, path, out, ws, ws_bytes, s);
  if (e == PFB_E_UNSUPPORTED && path != 1) return dual_path(g1, g2, 1, out, ws, ws_bytes, s);
  return e;
}

// ---------------------------------------------------------------------------
// Split-K partials (executor pass F15, gemm_parts.cu): for a skinny GEMM whose
// only consumers are fused elementwise groups, the k-splits write their
// partial tiles to parts[s] and the consumer sums them as it loads (split
// order, left to right), so the GEMM has no reduction phase.

static int parts_args(const pfb_tensor* a, const pfb_tensor* b, const pfb_tensor* out,
                      const void* b_planes, GemmArgs* g) {
  if (a->rank != 2 || b->rank != 2) return PFB_E_RANK;
  if (int e = matmul_args(a, b, const_cast<pfb_tensor*>(out), g)) return e;
  if (b_planes != nullptr) {
    g->b_hi = static_cast<const float*>(b_planes);
    g->b_lo = planes_lo(*g, b_planes);
  }
  return 0;
}

extern "C" int pfb_matmul_parts_count(const pfb_tensor* a, const pfb_tensor* b,
                                          const pfb_tensor* out) {
  static const bool off = getenv_flag("PFB_NO_PARTS");
  GemmArgs g;
  if (off || parts_args(a, b, out, nullptr, &g)) return 0;
  return gemm_parts_count(g);
}

extern "C" int64_t pfb_matmul_parts_workspace(const pfb_tensor* a, const pfb_tensor* b,
                                              const pfb_tensor* out) {
  GemmArgs g;
  if (parts_args(a, b, out, nullptr, &g)) return 0;
  return gemm_parts_workspace(g);
}

extern "C" int pfb_matmul_parts(const pfb_tensor* a, const pfb_tensor* b, pfb_tensor* parts,
                                const pfb_tensor* bias, const void* b_planes, void* ws,
                                int64_t ws_bytes, void* stream) {
  if (parts->rank != 3 || parts->dtype != PFB_F32 || parts->stride[2] != 1) return PFB_E_SHAPE;
  pfb_tensor out = *parts;
  out.rank = 2;
  out.shape[0] = parts->shape[1]; out.shape[1] = parts->shape[2];
  out.stride[0] = parts->stride[1]; out.stride[1] = parts->stride[2];
  GemmArgs g;
  if (int e = parts_args(a, b, &out, b_planes, &g)) return e;
  if (bias) {
    if (bias->dtype != PFB_F32) return PFB_E_DTYPE;
    int64_t st[2];
    if (!broadcast_strides(bias, 2, out.shape, st)) return PFB_E_SHAPE;
    g.bias = (const float*)bias->data;
    g.sxb = 0; g.sxm = st[0]; g.sxn = st[1];
  }
  const int S = gemm_parts_count(g);
  if (S < 1 || parts->shape[0] != S) return PFB_E_SHAPE;
  return gemm_parts(g, nullptr, S, (float*)parts->data, parts->stride[0], parts->stride[1], ws, ws_bytes,
                    as_stream(stream));
}

// Dual-operand form (a1 @ b1 + a2 @ b2, passes.fuse_dual_matmuls): the k-splits
// run over both K ranges back to back (cfg5's RNN cell x_t Wx + h Wh, whose
// row sums and select consume the partials).
static int dual_parts_args(const pfb_tensor* a1, const pfb_tensor* b1, const pfb_tensor* a2,
                           const pfb_tensor* b2, const pfb_tensor* out, const void* p1,
                           const void* p2, GemmArgs* g1, GemmArgs* g2) {
  if (int e = parts_args(a1, b1, out, p1, g1)) return e;
  return parts_args(a2, b2, out, p2, g2);
}

extern "C" int pfb_matmul_dual_parts_count(const pfb_tensor* a1, const pfb_tensor* b1,
                                           const pfb_tensor* a2, const pfb_tensor* b2,
                                           const pfb_tensor* out) {
  static const bool off = getenv_flag("PFB_NO_PARTS");
  GemmArgs g1, g2;
  if (off || dual_parts_args(a1, b1, a2, b2, out, nullptr, nullptr, &g1, &g2)) return 0;
  return gemm_parts_count(g1, &g2);
}

extern "C" int64_t pfb_matmul_dual_parts_workspace(const pfb_tensor* a1, const pfb_tensor* b1,
                                                   const pfb_tensor* a2, const pfb_tensor* b2,
                                                   const pfb_tensor* out) {
  GemmArgs g1, g2;
  if (dual_parts_args(a1, b1, a2, b2, out, nullptr, nullptr, &g1, &g2)) return 0;
  return gemm_parts_workspace(g1, &g2);
}

extern "C" int pfb_matmul_dual_parts(const pfb_tensor* a1, const pfb_tensor* b1,
                                     const pfb_tensor* a2, const pfb_tensor* b2,
                                     pfb_tensor* parts, const pfb_tensor* bias,
                                     const void* b1_planes, const void* b2_planes, void* ws,
                                     int64_t ws_bytes, void* stream) {
  if (parts->rank != 3 || parts->dtype != PFB_F32 || parts->stride[2] != 1) return PFB_E_SHAPE;
  pfb_tensor out = *parts;
  out.rank = 2;
  out.shape[0] = parts->shape[1]; out.shape[1] = parts->shape[2];
  out.stride[0] = parts->stride[1]; out.stride[1] = parts->stride[2];
  GemmArgs g1, g2;
  if (int e = dual_parts_args(a1, b1, a2, b2, &out, b1_planes, b2_planes, &g1, &g2)) return e;
  if (bias) {
    if (bias->dtype != PFB_F32) return PFB_E_DTYPE;
    int64_t st[2];
    if (!broadcast_strides(bias, 2, out.shape, st)) return PFB_E_SHAPE;
    g1.bias = (const float*)bias->data;
    g1.sxb = 0; g1.sxm = st[0]; g1.sxn = st[1];
  }
  const int S = gemm_parts_count(g1, &g2);
  if (S < 1 || parts->shape[0] != S) return PFB_E_SHAPE;
  return gemm_parts(g1, &g2, S, (float*)parts->data, parts->stride[0], parts->stride[1], ws,
                    ws_bytes, as_stream(stream));
}
