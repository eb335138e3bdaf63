// F2FP (cvt.rn.bf16x2.f32) throughput and its interaction with MUFU.EX2: 16 warps/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned* out, int iters, long long* cyc) {
  float a[8];
  unsigned r[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i * 1e-4f; r[i] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) {
        unsigned y;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        r[i] ^= y;
      }
      if (MODE == 1 || MODE == 2) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[(i + 4) & 7]));
      }
    }
  }
  long long t1 = clock64();
  unsigned s = 0;
  for (int i = 0; i < 8; ++i) s ^= r[i] ^ __float_as_uint(a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  unsigned* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int warps = 16, iters = 4096;
  const char* names[3] = {"F2FP only", "2x EX2 only", "F2FP + 2x EX2"};
  for (int mode = 0; mode < 3; ++mode) {
    if (mode == 0) k<0><<<148, warps * 32>>>(out, iters, cyc);
    if (mode == 1) k<1><<<148, warps * 32>>>(out, iters, cyc);
    if (mode == 2) k<2><<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double per_smsp_iters = double(warps) / 4 * 32 * 8 * iters;   // "units": one F2FP and/or two EX2 each
    printf("%-16s: %.2f clk per warp-instruction-group per SMSP (%.0f cycles)\n", names[mode],
           double(h) / (per_smsp_iters / 32), double(h));
  }
  return 0;
}
