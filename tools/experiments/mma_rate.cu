// Microbenchmark: issue rate of tcgen05.mma (cta_group::1, SS operands) by
// kind and N, one CTA per SM, all SMs busy.  Prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu && ./mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int KIND, bool VARY>  // 0 tf32, 1 bf16, 2 tf32 with A from TMEM
__global__ void __launch_bounds__(128, 1) bench(int n, uint32_t idesc, int iters, long long* out,
                                                int noise, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2[4];
  __shared__ uint32_t tslot;
  // pseudo-random operands (zeros let the tensor core run faster)
  for (int i = threadIdx.x; i < 80 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<float*>(smem)[i] = (float)(h & 0xffff) / 65536.f - 0.5f;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int j = 0; j < 4; ++j) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[j])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t da0 = desc_sw128(smem_u32(smem)), db0 = desc_sw128(smem_u32(smem + 32768));
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // VARY: walk 4 A and 4 B tiles (8 KB apart) and the 4 k-steps inside
      // each swizzle row, so no two consecutive MMAs read the same operands
      const uint64_t da = da0 + (VARY ? (uint64_t)(((i & 3) * 8192 + ((i >> 2) & 3) * 32) >> 4) : 0);
      const uint64_t db = db0 + (VARY ? (uint64_t)((((i >> 1) & 1) * 8192 + ((i >> 2) & 3) * 32) >> 4) : 0);
      if (mode && i % 12 == 0 && i > 0) {
        if (mode & 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(smem_u32(&bar2[(i / 12) & 3])) : "memory");
        if (mode & 2) asm volatile("tcgen05.fence::after_thread_sync;");
      }
      if (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(i));
      else if (KIND == 2)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                     ::"r"(tm), "r"(tm + 256 + (i & 3) * 8), "l"(db), "r"(idesc), "r"(i));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}"
                 ::"r"(smem_u32(&bar)) : "memory");
    t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  } else if (noise == 7 && threadIdx.x >= 32) {
    // 3 warps read TMEM (their lane quarter, 128 columns) in a loop: the
    // accumulator drain of a double-buffered TMEM tile
    const int q = (threadIdx.x >> 5) & 3;
    float s = 0.f;
    for (int r = 0; r < iters / 8; ++r) {
      for (int c = 0; c < 128; c += 32) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
            "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(tm + ((uint32_t)(q * 32) << 16) + 256 + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) s += __uint_as_float(v[j]);
      }
    }
    if (s == 12345.f) out[1] = 1;
  } else if (noise && noise != 7 && threadIdx.x >= 32) {
    // 3 warps stream 16 KB of shared memory (ld + st) while the MMAs run
    float4* q = reinterpret_cast<float4*>(smem + 65536);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < noise; ++r)
      for (int i = threadIdx.x - 32; i < 1024; i += 96) {
        float4 v = q[i];
        acc.x += v.x;
        q[i ^ 1] = acc;
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const int iters = 4096;
  for (int kind = 0; kind < 3; ++kind) {
    for (int n : {32, 64, 128, 256}) {
      if (kind == 2 && n == 256) continue;
      // c=f32 (1<<4); a/b format: tf32 = 2, bf16 = 1; N>>3 at 17; M>>4 at 24
      const uint32_t fmt = kind != 1 ? 2u : 1u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
     for (int vary = 0; vary < 2; ++vary) {
      auto k = vary ? (kind == 0 ? bench<0, true> : (kind == 1 ? bench<1, true> : bench<2, true>))
                    : (kind == 0 ? bench<0, false> : (kind == 1 ? bench<1, false> : bench<2, false>));
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
     for (int noise : {0, 1, 7, 8}) {
      k<<<148, 128, 80 * 1024>>>(n, idesc, iters, d, noise == 8 ? 7 : (noise == 7 ? 7 : 0), noise == 8 ? 1 : (noise == 7 ? 0 : noise));
      k<<<148, 128, 80 * 1024>>>(n, idesc, iters, d, noise == 8 ? 7 : (noise == 7 ? 7 : 0), noise == 8 ? 1 : (noise == 7 ? 0 : noise));
      cudaError_t e = cudaDeviceSynchronize();
      long long cyc = 0;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      const double kk = kind != 1 ? 8 : 16;
      const double per = (double)cyc / iters;
      printf("vary=%d mode=%d %s M=128 N=%3d K=%2.0f: %7.1f cycles/MMA  %7.1f flop/cycle/SM  (%s)\n", vary, noise,
             kind == 0 ? "tf32" : (kind == 1 ? "bf16" : "tf32 A-in-TMEM"), n, kk, per,
             2.0 * 128 * n * kk / per, cudaGetErrorString(e));
     }
     }
    }
  }
  return 0;
}
