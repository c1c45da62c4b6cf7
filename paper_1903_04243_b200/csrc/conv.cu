// Conv family, NHWC / HWIO, SAME padding, stride 1 (reference tensor.py:209-260).
//
// The configs' convolutions are tiny-channel (3x3x1x8 on 28x28 MNIST
// images), so the direct form -- one thread per output pixel x channel, the
// k1*k2*c1 window read from L1/L2 -- is HBM-bound on the image and needs no
// im2col buffer.  conv2d_input_grad is the exact adjoint (col2im gather form:
// each input pixel sums the window positions that read it), so no atomics.
#include "common.cuh"

namespace pfb {

struct ConvDims {
  int64_t b, h, w, c1, c2;
  int k1, k2, p1, p2;  // SAME: p = floor((k-1)/2) before
};

// x/out/f must be dense (executor materialises views first)
__global__ void conv2d_direct(ConvDims d, const float* __restrict__ x, const float* __restrict__ f,
                              float* __restrict__ out) {
  pdl_enter();
  const int64_t total = d.b * d.h * d.w * d.c2;
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < total;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int64_t co = lin % d.c2;
    int64_t t = lin / d.c2;
    int64_t j = t % d.w; t /= d.w;
    int64_t i = t % d.h;
    int64_t bb = t / d.h;
    float acc = 0.f;
    for (int p = 0; p < d.k1; ++p) {
      int64_t ii = i + p - d.p1;
      if (ii < 0 || ii >= d.h) continue;
      for (int q = 0; q < d.k2; ++q) {
        int64_t jj = j + q - d.p2;
        if (jj < 0 || jj >= d.w) continue;
        const float* xp = x + ((bb * d.h + ii) * d.w + jj) * d.c1;
        const float* fp = f + ((int64_t)(p * d.k2 + q) * d.c1) * d.c2 + co;
        for (int64_t c = 0; c < d.c1; ++c) acc = fmaf(__ldg(xp + c), __ldg(fp + c * d.c2), acc);
      }
    }
    out[lin] = acc;
  }
}

__global__ void conv2d_input_grad_direct(ConvDims d, const float* __restrict__ gy,
                                         const float* __restrict__ f, float* __restrict__ dx) {
  pdl_enter();
  const int64_t total = d.b * d.h * d.w * d.c1;
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < total;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int64_t ci = lin % d.c1;
    int64_t t = lin / d.c1;
    int64_t j = t % d.w; t /= d.w;
    int64_t i = t % d.h;
    int64_t bb = t / d.h;
    float acc = 0.f;
    // output pixel (oi, oj) reads input (oi + p - p1, oj + q - p2)
    for (int p = 0; p < d.k1; ++p) {
      int64_t oi = i - p + d.p1;
      if (oi < 0 || oi >= d.h) continue;
      for (int q = 0; q < d.k2; ++q) {
        int64_t oj = j - q + d.p2;
        if (oj < 0 || oj >= d.w) continue;
        const float* gp = gy + ((bb * d.h + oi) * d.w + oj) * d.c2;
        const float* fp = f + ((int64_t)(p * d.k2 + q) * d.c1 + ci) * d.c2;
        for (int64_t c = 0; c < d.c2; ++c) acc = fmaf(__ldg(gp + c), __ldg(fp + c), acc);
      }
    }
    dx[lin] = acc;
  }
}

__global__ void im2col_kernel(ConvDims d, const float* __restrict__ x, float* __restrict__ cols) {
  pdl_enter();
  const int64_t kc = (int64_t)d.k1 * d.k2 * d.c1;
  const int64_t total = d.b * d.h * d.w * kc;
  for (int64_t lin = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; lin < total;
       lin += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = lin % kc;
    int64_t pix = lin / kc;
    int64_t c = e % d.c1;
    int64_t pq = e / d.c1;
    int q = (int)(pq % d.k2), p = (int)(pq / d.k2);
    int64_t j = pix % d.w;
    int64_t t = pix / d.w;
    int64_t i = t % d.h;
    int64_t bb = t / d.h;
    int64_t ii = i + p - d.p1, jj = j + q - d.p2;
    float v = 0.f;
    if (ii >= 0 && ii < d.h && jj >= 0 && jj < d.w) v = __ldg(x + ((bb * d.h + ii) * d.w + jj) * d.c1 + c);
    cols[lin] = v;
  }
}

inline void same_pad(int k, int* before) { *before = (k - 1) / 2; }

// ---------------------------------------------------------------------------
// Per-example tiled kernels: one CTA per example, the zero-padded image in
// shared memory (SAME halo), the k1*k2*c window of each output pixel read from
// there.  KC = k1*k2*c1 and O = c2 are compile-time (small-channel configs:
// the MNIST ConvNet is 3x3x1x8); other shapes use the direct kernels above.

template <int KC, int O>
__device__ __forceinline__ void window(const float* xs, int wp, int c1, int k2, int i, int j,
                                       float (&xv)[KC]) {
#pragma unroll
  for (int e = 0; e < KC; ++e) {
    const int c = e % c1, pq = e / c1;
    const int q = pq % k2, p = pq / k2;
    xv[e] = xs[((i + p) * wp + (j + q)) * c1 + c];
  }
}

__device__ __forceinline__ void stage_image(const float* __restrict__ x, float* xs, int h, int w,
                                            int c1, int p1, int p2, int hp, int wp) {
  for (int t = threadIdx.x; t < hp * wp * c1; t += blockDim.x) {
    const int c = t % c1, pix = t / c1;
    const int jj = pix % wp - p2, ii = pix / wp - p1;
    xs[t] = (ii >= 0 && ii < h && jj >= 0 && jj < w) ? __ldg(x + ((int64_t)ii * w + jj) * c1 + c)
                                                     : 0.f;
  }
}

// out[b][pix][o] = sum_e window(b, pix)[e] * f[e][o]  (reference tensor.py:232-241)
template <int KC, int O>
__global__ void __launch_bounds__(256) conv2d_tiled(ConvDims d, const float* __restrict__ x,
                                                    const float* __restrict__ f,
                                                    float* __restrict__ out) {
  extern __shared__ float sm[];
  pdl_enter();
  const int h = (int)d.h, w = (int)d.w, c1 = (int)d.c1;
  const int hp = h + d.k1 - 1, wp = w + d.k2 - 1;
  float* fs = sm;               // [KC][O]
  float* xs = sm + KC * O;      // [hp][wp][c1]
  const int64_t b = blockIdx.x;
  for (int t = threadIdx.x; t < KC * O; t += blockDim.x) fs[t] = __ldg(f + t);
  stage_image(x + b * h * w * c1, xs, h, w, c1, d.p1, d.p2, hp, wp);
  __syncthreads();
  float* ob = out + b * h * w * O;
  for (int pix = threadIdx.x; pix < h * w; pix += blockDim.x) {
    float xv[KC];
    window<KC, O>(xs, wp, c1, d.k2, pix / w, pix % w, xv);
    float acc[O];
#pragma unroll
    for (int o = 0; o < O; ++o) acc[o] = 0.f;
#pragma unroll
    for (int e = 0; e < KC; ++e)
#pragma unroll
      for (int o = 0; o < O; ++o) acc[o] = fmaf(xv[e], fs[e * O + o], acc[o]);
    if constexpr (O % 4 == 0) {
#pragma unroll
      for (int o = 0; o < O; o += 4)
        *reinterpret_cast<float4*>(ob + (int64_t)pix * O + o) =
            make_float4(acc[o], acc[o + 1], acc[o + 2], acc[o + 3]);
    } else {
#pragma unroll
      for (int o = 0; o < O; ++o) ob[(int64_t)pix * O + o] = acc[o];
    }
  }
}

// Per-example filter gradient (the conv2d VJP w.r.t. the filter, reference
// autodiff.py over tensor.py:209-229: im2col(x_b)^T gy_b) without the im2col
// buffer: every thread accumulates the KC x O products of its pixels in
// registers, then a fixed-order warp-shuffle + shared-memory tree sums them
// (deterministic).  out[b][e][o]; sq_norm[b] (nullable) = sum of squares of
// that block (the per-example norm term of F1).
template <int KC, int O>
__global__ void __launch_bounds__(256) conv2d_filter_grad_tiled(
    ConvDims d, const float* __restrict__ x, const float* __restrict__ gy, float* __restrict__ out,
    float* __restrict__ sq_norm) {
  extern __shared__ float sm[];
  __shared__ float part[8][KC * O];
  pdl_enter();
  const int h = (int)d.h, w = (int)d.w, c1 = (int)d.c1;
  const int hp = h + d.k1 - 1, wp = w + d.k2 - 1;
  float* xs = sm;
  const int64_t b = blockIdx.x;
  stage_image(x + b * h * w * c1, xs, h, w, c1, d.p1, d.p2, hp, wp);
  __syncthreads();
  const float* gb = gy + b * h * w * O;
  float acc[KC * O];
#pragma unroll
  for (int e = 0; e < KC * O; ++e) acc[e] = 0.f;
  for (int pix = threadIdx.x; pix < h * w; pix += blockDim.x) {
    float xv[KC];
    window<KC, O>(xs, wp, c1, d.k2, pix / w, pix % w, xv);
    float g[O];
    if constexpr (O % 4 == 0) {
#pragma unroll
      for (int o = 0; o < O; o += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(gb + (int64_t)pix * O + o));
        g[o] = v.x; g[o + 1] = v.y; g[o + 2] = v.z; g[o + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int o = 0; o < O; ++o) g[o] = __ldg(gb + (int64_t)pix * O + o);
    }
#pragma unroll
    for (int e = 0; e < KC; ++e)
#pragma unroll
      for (int o = 0; o < O; ++o) acc[e * O + o] = fmaf(xv[e], g[o], acc[e * O + o]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < KC * O; ++e) {
    float v = acc[e];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) part[warp][e] = v;
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float sq = 0.f;
  for (int e = threadIdx.x; e < KC * O; e += blockDim.x) {
    float v = part[0][e];
    for (int q = 1; q < nw; ++q) v += part[q][e];
    out[b * KC * O + e] = v;
    sq = fmaf(v, v, sq);
  }
  if (sq_norm != nullptr) {  // KC*O <= blockDim: one value per thread, tree over the block
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    __syncthreads();
    if (lane == 0) part[0][warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int q = 0; q < nw; ++q) t += part[0][q];
      sq_norm[b] = t;
    }
  }
}

// (KC, O) pairs with tiled kernels; anything else -> the direct / im2col forms
#define PFB_CONV_SHAPES(X) X(9, 8) X(9, 16) X(9, 4) X(27, 8) X(25, 8) X(9, 1)
// filter gradients keep KC x O accumulators per thread: <= 128
#define PFB_FGRAD_SHAPES(X) X(9, 8) X(9, 4) X(9, 1) X(9, 12) X(25, 4) X(27, 4)

template <int KC, int O>
static bool conv_tiled_launch(const ConvDims& d, const float* x, const float* f, float* out,
                              cudaStream_t s) {
  const int64_t smem = (int64_t)(KC * O + (d.h + d.k1 - 1) * (d.w + d.k2 - 1) * d.c1) * 4;
  if (smem > 160 * 1024) return false;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv2d_tiled<KC, O>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         160 * 1024);
    attr = true;
  }
  launch(conv2d_tiled<KC, O>, (int)d.b, 256, (size_t)smem, s, d, x, f, out);
  return true;
}

template <int KC, int O>
static bool filter_grad_tiled_launch(const ConvDims& d, const float* x, const float* gy,
                                     float* out, float* sq, cudaStream_t s) {
  const int64_t smem = (int64_t)((d.h + d.k1 - 1) * (d.w + d.k2 - 1) * d.c1) * 4;
  if (smem > 160 * 1024 || KC * O > 128) return false;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv2d_filter_grad_tiled<KC, O>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  launch(conv2d_filter_grad_tiled<KC, O>, (int)d.b, 256, (size_t)smem, s, d, x, gy, out, sq);
  return true;
}

}  // namespace pfb

using namespace pfb;

extern "C" int pfb_im2col(const pfb_tensor* x, int32_t k1, int32_t k2, pfb_tensor* out, void* stream) {
  if (x->rank != 4) return PFB_E_RANK;
  if (x->dtype != PFB_F32 || out->dtype != PFB_F32) return PFB_E_DTYPE;
  if (!is_dense(x) || !is_dense(out)) return PFB_E_UNSUPPORTED;
  ConvDims d{x->shape[0], x->shape[1], x->shape[2], x->shape[3], 0, k1, k2, 0, 0};
  same_pad(k1, &d.p1);
  same_pad(k2, &d.p2);
  int64_t n = d.b * d.h * d.w * k1 * k2 * d.c1;
  if (n == 0) return 0;
  launch(im2col_kernel, grid_for(n, 256), 256, 0, as_stream(stream), d, (const float*)x->data,
                                                                 (float*)out->data);
  return launch_status();
}

extern "C" int pfb_conv2d(const pfb_tensor* x, const pfb_tensor* f, pfb_tensor* out, void* stream) {
  if (x->rank != 4 || f->rank != 4) return PFB_E_RANK;
  if (x->dtype != PFB_F32 || f->dtype != PFB_F32) return PFB_E_DTYPE;
  if (x->shape[3] != f->shape[2]) return PFB_E_SHAPE;
  if (!is_dense(x) || !is_dense(f) || !is_dense(out)) return PFB_E_UNSUPPORTED;
  ConvDims d{x->shape[0], x->shape[1], x->shape[2], x->shape[3], f->shape[3],
             (int)f->shape[0], (int)f->shape[1], 0, 0};
  same_pad(d.k1, &d.p1);
  same_pad(d.k2, &d.p2);
  int64_t n = d.b * d.h * d.w * d.c2;
  if (n == 0) return 0;
  const int kc = d.k1 * d.k2 * (int)d.c1;
  bool done = false;
#define PFB_TRY_CONV(KC_, O_)                                                                   \
  if (!done && kc == KC_ && d.c2 == O_ && d.b <= 2147483647)                                     \
    done = conv_tiled_launch<KC_, O_>(d, (const float*)x->data, (const float*)f->data,          \
                                      (float*)out->data, as_stream(stream));
  PFB_CONV_SHAPES(PFB_TRY_CONV)
#undef PFB_TRY_CONV
  if (done) return launch_status();
  launch(conv2d_direct, grid_for(n, 256), 256, 0, as_stream(stream), d, (const float*)x->data,
                                                                 (const float*)f->data,
                                                                 (float*)out->data);
  return launch_status();
}

extern "C" int pfb_conv2d_input_grad(const pfb_tensor* gy, const pfb_tensor* f, pfb_tensor* out,
                                     void* stream) {
  if (gy->rank != 4 || f->rank != 4) return PFB_E_RANK;
  if (gy->dtype != PFB_F32 || f->dtype != PFB_F32) return PFB_E_DTYPE;
  if (gy->shape[3] != f->shape[3]) return PFB_E_SHAPE;
  if (!is_dense(gy) || !is_dense(f) || !is_dense(out)) return PFB_E_UNSUPPORTED;
  ConvDims d{gy->shape[0], gy->shape[1], gy->shape[2], f->shape[2], gy->shape[3],
             (int)f->shape[0], (int)f->shape[1], 0, 0};
  same_pad(d.k1, &d.p1);
  same_pad(d.k2, &d.p2);
  int64_t n = d.b * d.h * d.w * d.c1;
  if (n == 0) return 0;
  launch(conv2d_input_grad_direct, grid_for(n, 256), 256, 0, as_stream(stream), 
      d, (const float*)gy->data, (const float*)f->data, (float*)out->data);
  return launch_status();
}

// per-example filter gradient (passes.fuse_conv_filter_grads):
//   out[b, (p*k2+q)*c1+c, o] = sum_{i,j} x[b, i+p-p1, j+q-p2, c] gy[b, i, j, o]
// x [b,h,w,c1], gy [b,h,w,c2] dense; out [b, k1*k2*c1, c2]; sq_norm (nullable)
// [b] = sum of squares of out[b].  PFB_E_UNSUPPORTED for shapes without a
// tiled kernel (the executor then runs im2col + batched GEMM).
extern "C" int pfb_conv2d_filter_grad(const pfb_tensor* x, const pfb_tensor* gy, int32_t k1,
                                      int32_t k2, pfb_tensor* out, pfb_tensor* sq_norm,
                                      void* stream) {
  if (x->rank != 4 || gy->rank != 4 || out->rank != 3) return PFB_E_RANK;
  if (x->dtype != PFB_F32 || gy->dtype != PFB_F32 || out->dtype != PFB_F32) return PFB_E_DTYPE;
  for (int i = 0; i < 3; ++i)
    if (x->shape[i] != gy->shape[i]) return PFB_E_SHAPE;
  if (out->shape[0] != x->shape[0] || out->shape[1] != (int64_t)k1 * k2 * x->shape[3] ||
      out->shape[2] != gy->shape[3])
    return PFB_E_SHAPE;
  if (sq_norm && (sq_norm->rank != 1 || sq_norm->shape[0] != x->shape[0] || !is_dense(sq_norm)))
    return PFB_E_SHAPE;
  if (!is_dense(x) || !is_dense(gy) || !is_dense(out)) return PFB_E_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(gy->data) & 15) != 0) return PFB_E_UNSUPPORTED;
  ConvDims d{x->shape[0], x->shape[1], x->shape[2], x->shape[3], gy->shape[3], k1, k2, 0, 0};
  same_pad(k1, &d.p1);
  same_pad(k2, &d.p2);
  if (d.b == 0) return 0;
  const int kc = k1 * k2 * (int)d.c1;
  bool done = false;
#define PFB_TRY_FG(KC_, O_)                                                                     \
  if (!done && kc == KC_ && d.c2 == O_ && d.b <= 2147483647)                                     \
    done = filter_grad_tiled_launch<KC_, O_>(d, (const float*)x->data, (const float*)gy->data,  \
                                             (float*)out->data,                                 \
                                             sq_norm ? (float*)sq_norm->data : nullptr,         \
                                             as_stream(stream));
  PFB_FGRAD_SHAPES(PFB_TRY_FG)
#undef PFB_TRY_FG
  return done ? launch_status() : PFB_E_UNSUPPORTED;
}
