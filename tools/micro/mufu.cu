// MUFU.EX2 throughput probe: W warps per SM, each lane runs 8 independent ex2 chains; cycles per ex2 per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 4096;
    k<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double exps_per_smsp = double(warps) / 4 * 32 * 8 * iters;
    printf("warps/SM %2d: %.2f ex2 per clk per SMSP (%.0f cycles)\n", warps, exps_per_smsp / h[0], double(h[0]));
  }
  return 0;
}
