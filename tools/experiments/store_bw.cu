// Microbenchmark: HBM write bandwidth of the GEMM epilogue store paths, one
// CTA per SM (persistent), 8 store warps, 2 GiB output:
//   mode 0: TMA store, box {32 cols, 32 rows} (4 KB, per warp)     -- current epilogues
//   mode 1: TMA store, box {32 cols, 128 rows} (16 KB, 4 warps)
//   mode 2: TMA store, 3-D box {32 cols, 128 rows, 4 col-blocks} (64 KB, 8 warps... 2 halves)
//   mode 3: st.global.v4 through a smem transpose (4 rows x 128 B per warp instruction)
//   mode 4: st.global.v4 straight from registers (lane = row: 32 rows x 16 B per instruction)
// Measured (profiles/r02/README.md): modes 0-3 5.9-6.1 TB/s, mode 4 1.5 TB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_bw store_bw.cu -lcuda && ./store_bw
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int M = 32768, N = 16384;  // 2 GiB fp32
constexpr int TM = 128, TN = 128;    // output tile per CTA iteration

__global__ void __launch_bounds__(256, 1) store_kernel(const __grid_constant__ CUtensorMap m32,
                                                        const __grid_constant__ CUtensorMap m128,
                                                        const __grid_constant__ CUtensorMap m3d,
                                                        float* C, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* smem = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, half = warp >> 2;  // rows quarter*32.., cols half*64..
  const int tiles = (M / TM) * (N / TN);
  // staging: 2 buffers x [4 col-blocks][128 rows][32 cols] = 2 x 64 KB
  int buf = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x, buf ^= 1) {
    const int m0 = (t / (N / TN)) * TM, n0 = (t % (N / TN)) * TN;
    float* st = smem + buf * (TM * TN);
    if (mode == 4) {
      // registers -> global, no shared memory: lane = row, 32 consecutive columns
      // per lane as 8 x 16-byte stores (each warp instruction: 32 rows x 16 B)
      for (int cb = 0; cb < 2; ++cb) {
        const int col0 = n0 + half * 64 + cb * 32;
        float* rowp = C + (int64_t)(m0 + quarter * 32 + lane) * N + col0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(rowp + 4 * q) = make_float4(t, q, cb, lane);
      }
      continue;
    }
    if (mode == 3) {
      // registers -> smem transpose -> 4-row x 128-byte stores
      float* blk = smem + warp * 1024;
      for (int cb = 0; cb < 2; ++cb) {
        const int col0 = n0 + half * 64 + cb * 32;
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(blk + lane * 32 + 4 * (q ^ (lane & 7))) =
              make_float4(t, q, cb, lane);
        __syncwarp();
        const int sub_r = lane >> 3, sub_c = (lane & 7) * 4;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const int srow = i + sub_r;
          const float4 w = *reinterpret_cast<const float4*>(blk + srow * 32 + 4 * ((sub_c >> 2) ^ (srow & 7)));
          *reinterpret_cast<float4*>(C + (int64_t)(m0 + quarter * 32 + srow) * N + col0 + sub_c) = w;
        }
        __syncwarp();
      }
      continue;
    }
    // wait until the stores that last read this buffer are done (per issuing thread)
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    for (int cb = 0; cb < 2; ++cb) {
      const int cblk = half * 2 + cb;  // 32-col block 0..3
      float* blk = st + cblk * (TM * 32) + quarter * 32 * 32;
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(blk + lane * 32 + 4 * (q ^ (lane & 7))) = make_float4(t, q, cb, lane);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (mode == 0 && lane == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                     ::"l"(&m32), "r"(smem_u32(blk)), "r"(n0 + cblk * 32), "r"(m0 + quarter * 32) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (mode == 1 || mode == 2) {
      __syncthreads();
      if (mode == 1 && lane == 0 && quarter == 0) {
        for (int cb = 0; cb < 2; ++cb) {
          const int cblk = half * 2 + cb;
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                       ::"l"(&m128), "r"(smem_u32(st + cblk * TM * 32)), "r"(n0 + cblk * 32), "r"(m0) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (mode == 2 && threadIdx.x == 0) {
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                     ::"l"(&m3d), "r"(smem_u32(st)), "r"(0), "r"(m0), "r"(n0 / 32) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  float* C;
  cudaMalloc(&C, (size_t)M * N * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m32, m128, m3d;
  cuuint64_t dims[2] = {N, M};
  cuuint64_t strides[1] = {(cuuint64_t)N * 4};
  cuuint32_t estr[3] = {1, 1, 1};
  cuuint32_t box32[2] = {32, 32}, box128[2] = {32, 128};
  enc(&m32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box32, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m128, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box128, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d3[3] = {32, M, N / 32};
  cuuint64_t s3[2] = {(cuuint64_t)N * 4, 128};
  cuuint32_t b3[3] = {32, 128, 4};
  CUresult r = enc(&m3d, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, C, d3, s3, b3, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("3d map encode: %d\n", (int)r);
  const int smem = 2 * TM * TN * 4 + 1024;
  cudaFuncSetAttribute(store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[5] = {"TMA box 32x32 (4 KB/warp)", "TMA box 32x128 (16 KB)", "TMA 3-D box 32x128x4 (64 KB)",
                          "st.global.v4 via smem transpose", "st.global.v4 from registers (row/lane)"};
  for (int mode = 0; mode < 5; ++mode) {
    if (mode == 2 && r != CUDA_SUCCESS) continue;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    store_kernel<<<sms, 256, smem>>>(m32, m128, m3d, C, mode);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) store_kernel<<<sms, 256, smem>>>(m32, m128, m3d, C, mode);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("mode %d %-34s: %7.0f GB/s (%s)\n", mode, names[mode], 5.0 * M * N * 4 / (ms / 1e3) / 1e9,
           cudaGetErrorString(e));
  }
  return 0;
}
