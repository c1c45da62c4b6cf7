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
