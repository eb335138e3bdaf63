// TMEM load / store throughput on one SM: W warps (W/4 per lane quarter) repeatedly read (or write) their 32 lanes
// x C columns with tcgen05.ld/st.32x32b.x32 (and the 16x256b.x8 shape), clock64 around the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_09741_b200/csrc -I include \
//        tools/micro/tmem_bw.cu -o /tmp/tmem_bw && /tmp/tmem_bw
#include <cstdio>

#include "common.cuh"
#include "ptx.cuh"

using namespace tp;

template <int MODE>   // 0: ld 32x32b.x32, 1: st 32x32b.x32, 2: ld 16x256b.x8
__global__ void tmem_bw_kernel(int iters, int cols_per_warp, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int q = warp & 3, g = warp >> 2;   // lane quarter, column group of this warp
  const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16) + g * cols_per_warp;
  uint32_t acc = 0;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < cols_per_warp; c += 32) {
      if (MODE == 0) {
        tmem_ld32(base + c, r);
        tmem_wait_ld();
        acc += r[0] ^ r[13] ^ r[31];
      } else if (MODE == 1) {
        tmem_st32(base + c, r);
        tmem_wait_st();
      } else {
        tmem_ld_16x256b_x8(base + c + ((threadIdx.x & 32) ? 0 : 0), r);   // 16 lanes x 64 columns
        tmem_wait_ld();
        acc += r[0] ^ r[13] ^ r[31];
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0xdeadbeef) *sink = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d_out;
  uint32_t* sink;
  cudaMalloc(&d_out, 8 * 256);
  cudaMalloc(&sink, 4);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16}) {
      const int cols_per_warp = 128 * 4 / warps;   // the warps of one quarter together cover 128 columns
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) tmem_bw_kernel<0><<<1, warps * 32>>>(iters, cols_per_warp, d_out, sink);
        if (mode == 1) tmem_bw_kernel<1><<<1, warps * 32>>>(iters, cols_per_warp, d_out, sink);
        if (mode == 2) tmem_bw_kernel<2><<<1, warps * 32>>>(iters, cols_per_warp, d_out, sink);
      }
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long cyc = 0;
      cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
      const double bytes = 128.0 * 128 * 4 * iters;   // every mode reads or writes 128 lanes x 128 columns per iteration
      std::printf("mode %s warps %2d: %.1f B/cycle (%s)\n", mode == 0 ? "ld32x32b" : mode == 1 ? "st32x32b" : "ld16x256b",
                  warps, bytes / cyc, cudaGetErrorString(e));
    }
  }
  return 0;
}
