// The forward softmax's exp pass in isolation: 1 warp per SMSP (4 warps/SM), 128 fp32 values per thread in
// registers, per pair FFMA2 -> 2x MUFU.EX2 -> FADD2 (4 chains) + F2FP; cycles per 128-element pass.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 a) {
  return (static_cast<unsigned long long>(__float_as_uint(a.y)) << 32) | __float_as_uint(a.x);
}
__device__ __forceinline__ float2 u2f(unsigned long long r) {
  return make_float2(__uint_as_float(static_cast<unsigned>(r)), __uint_as_float(static_cast<unsigned>(r >> 32)));
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pack(float a, float b) { unsigned r; asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r; }

template <bool SEPARATE>
__global__ void k(unsigned* out, int iters, long long* cyc, float sc, float m) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = (threadIdx.x + i) * 1e-3f;
  unsigned acc = 0;
  float2 tot = make_float2(0.f, 0.f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float2 sa2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    const float2 sc2 = make_float2(sc, sc), nm2 = make_float2(-m - it * 1e-7f, -m);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      unsigned pw[16];
      if (SEPARATE) {
        float p[32];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 a2 = ffma2(make_float2(s[c * 32 + i], s[c * 32 + i + 1]), sc2, nm2);
          p[i] = ex2(a2.x);
          p[i + 1] = ex2(a2.y);
        }
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          sa2[(i >> 1) & 3] = fadd2(sa2[(i >> 1) & 3], make_float2(p[i], p[i + 1]));
          pw[i / 2] = pack(p[i], p[i + 1]);
        }
      } else {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float2 a2 = ffma2(make_float2(s[c * 32 + i], s[c * 32 + i + 1]), sc2, nm2);
        const float p0 = ex2(a2.x), p1 = ex2(a2.y);
        sa2[(i >> 1) & 3] = fadd2(sa2[(i >> 1) & 3], make_float2(p0, p1));
        pw[i / 2] = pack(p0, p1);
      }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc ^= pw[i];
    }
    tot = fadd2(tot, fadd2(fadd2(sa2[0], sa2[1]), fadd2(sa2[2], sa2[3])));
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(tot.x + tot.y);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  unsigned* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int sep = 0; sep < 2; ++sep)
  for (int warps : {4, 8}) {
    const int iters = 2000;
    if (sep) k<true><<<148, warps * 32>>>(out, iters, cyc, 0.1f, 1.0f);
    else k<false><<<148, warps * 32>>>(out, iters, cyc, 0.1f, 1.0f);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("separate %d warps/SM %d: %.0f cycles per 128-element pass per warp-slot (MUFU floor %d)\n", sep, warps,
           double(h) / iters, warps / 4 * 1024);
  }
  return 0;
}
