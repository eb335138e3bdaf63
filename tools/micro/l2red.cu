// L2 fp32 reduction throughput: red.global.add.v4.f32 (row-per-thread and coalesced) vs TMA reduce-add.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2511_09741_b200/csrc/ptx.cuh"
using namespace tp;

__global__ void red_rowwise(float* dst, int iters, int ntiles, int H) {
  // tile = 128 rows x 128 fp32; thread t owns row t (like the dQ warps), 32 x red.v4
  const int t = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const int tile = (blockIdx.x + it * gridDim.x) % ntiles;
    float* row = dst + (size_t)(tile * 128 + t) * H;
#pragma unroll 4
    for (int v = 0; v < 32; ++v)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + v * 4), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
  }
}
__global__ void red_coalesced(float* dst, int iters, int ntiles, int H) {
  const int t = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const int tile = (blockIdx.x + it * gridDim.x) % ntiles;
#pragma unroll 4
    for (int v = 0; v < 32; ++v) {
      const int e = v * 128 + t;         // 4096 float4 per tile; consecutive threads -> consecutive 16 B
      const int r = e / 32, c = (e % 32) * 4;
      float* p = dst + (size_t)(tile * 128 + r) * H + c;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
    }
  }
}
// 16x256b-like pattern: thread t -> row (t/4) (+8), 2 consecutive columns at 2*(t%4): 4 threads = one 32 B sector
__global__ void red_sector_v2(float* dst, int iters, int ntiles, int H) {
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;  // 4 warps, warp w owns rows [32w, 32w+32)
  for (int it = 0; it < iters; ++it) {
    const int tile = (blockIdx.x + it * gridDim.x) % ntiles;
#pragma unroll 4
    for (int half = 0; half < 2; ++half)
      for (int cg = 0; cg < 16; ++cg)
        for (int rr = 0; rr < 2; ++rr) {
          const int row = w * 32 + half * 16 + rr * 8 + lane / 4;
          float* p = dst + (size_t)(tile * 128 + row) * H + cg * 8 + (lane % 4) * 2;
          asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(1.f) : "memory");
        }
  }
}
// 2 threads x 16 B = 32 B per row, 16 rows per warp instruction
__global__ void red_sector_v4(float* dst, int iters, int ntiles, int H) {
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  for (int it = 0; it < iters; ++it) {
    const int tile = (blockIdx.x + it * gridDim.x) % ntiles;
#pragma unroll 4
    for (int half = 0; half < 2; ++half)
      for (int cg = 0; cg < 16; ++cg) {
        const int row = w * 32 + half * 16 + lane / 2;
        float* p = dst + (size_t)(tile * 128 + row) * H + cg * 8 + (lane % 2) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
  }
}
__global__ void tma_red(const __grid_constant__ CUtensorMap tm, int iters, int ntiles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 65536 / 4; ++i) reinterpret_cast<float*>(sm)[i] = 1.f;
    fence_async_smem_dummy:;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int it = 0; it < iters; ++it) {
      const int tile = (blockIdx.x + it * gridDim.x) % ntiles;
      for (int c = 0; c < 4; ++c) tma_reduce_add_2d(&tm, sm + c * 16384, c * 32, tile * 128);
      bulk_commit();
      if (it >= 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    bulk_wait_all0();
  }
}

int main() {
  const int H = 128, ntiles = 256, iters = 200;
  float* d; cudaMalloc(&d, (size_t)ntiles * 128 * H * 4); cudaMemset(d, 0, (size_t)ntiles * 128 * H * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = 148.0 * iters * 65536;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); red_rowwise<<<148, 128>>>(d, iters, ntiles, H); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("red.v4 row-per-thread : %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(a); red_coalesced<<<148, 128>>>(d, iters, ntiles, H); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("red.v4 coalesced      : %.1f GB/s\n", bytes / ms / 1e6);
    // 296 CTAs (2 per SM) variants
    cudaEventRecord(a); red_coalesced<<<296, 128>>>(d, iters / 2, ntiles, H); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("red.v4 coalesced x2   : %.1f GB/s\n", bytes / ms / 1e6);
  }
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); red_sector_v2<<<148, 128>>>(d, iters, ntiles, H); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("red.v2 sector (16x256b): %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(a); red_sector_v4<<<148, 128>>>(d, iters, ntiles, H); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("red.v4 sector pairs   : %.1f GB/s\n", bytes / ms / 1e6);
  }
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", (void**)&enc, 12000, cudaEnableDefault, &q);
  CUtensorMap tm; cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)ntiles * 128}; cuuint64_t str[1] = {(cuuint64_t)H * 4};
  cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(tma_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); tma_red<<<148, 32, 65536>>>(tm, iters, ntiles); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("TMA reduce-add        : %.1f GB/s (%s)\n", bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
