// Which instruction in the softmax exp pass costs MUFU throughput?  1 warp per SMSP, 128 values per thread.
// variant 0: FFMA2 + 2 EX2 + FADD2 + F2FP (the kernel's mix); 1: no F2FP; 2: no FADD2; 3: EX2 only (+FFMA2)
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
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pack(float a, float b) { unsigned r; asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r; }
// integer packs on the ALU pipe: round half up (one add per value) / round to nearest even
__device__ __forceinline__ unsigned pack_hu(float a, float b) {
  const unsigned ua = __float_as_uint(a) + 0x8000u, ub = __float_as_uint(b) + 0x8000u;
  return __byte_perm(ua, ub, 0x7632);
}
__device__ __forceinline__ unsigned pack_rne(float a, float b) {
  unsigned ua = __float_as_uint(a), ub = __float_as_uint(b);
  ua += 0x7FFFu + ((ua >> 16) & 1u);
  ub += 0x7FFFu + ((ub >> 16) & 1u);
  return __byte_perm(ua, ub, 0x7632);
}

template <int V>
__global__ void k(unsigned* out, int iters, long long* cyc) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = (threadIdx.x + i) * 1e-3f;
  unsigned acc[16] = {0};
  float2 sa2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float2 sc2 = make_float2(0.1f, 0.1f), nm2 = make_float2(-1.f - it * 1e-7f, -1.f);
#pragma unroll
    for (int i = 0; i < 128; i += 2) {
      const float2 a2 = ffma2(make_float2(s[i], s[i + 1]), sc2, nm2);
      const float p0 = ex2(a2.x), p1 = ex2(a2.y);
      if (V == 0 || V == 1) sa2[(i >> 1) & 3] = fadd2(sa2[(i >> 1) & 3], make_float2(p0, p1));
      if (V == 0 || V == 2) acc[(i >> 1) & 15] ^= pack(p0, p1);
      if (V == 4 || V == 5) sa2[(i >> 1) & 3] = fadd2(sa2[(i >> 1) & 3], make_float2(p0, p1));
      if (V == 4) acc[(i >> 1) & 15] ^= pack_hu(p0, p1);
      if (V == 5) acc[(i >> 1) & 15] ^= pack_rne(p0, p1);
      if (V == 3) acc[(i >> 1) & 15] ^= __float_as_uint(p0) ^ __float_as_uint(p1);
      if (V == 2) acc[(i >> 2) & 15] += __float_as_uint(p0);
    }
  }
  long long t1 = clock64();
  unsigned r = __float_as_uint(sa2[0].x + sa2[1].y + sa2[2].x + sa2[3].y);
  for (int i = 0; i < 16; ++i) r ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  unsigned* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[6] = {"FFMA2+2EX2+FADD2+F2FP", "no F2FP", "no FADD2", "EX2 + XOR only", "int pack half-up",
                          "int pack RNE"};
  for (int v = 0; v < 6; ++v)
    for (int warps : {4, 8}) {
      const int iters = 2000;
      if (v == 0) k<0><<<148, warps * 32>>>(out, iters, cyc);
      if (v == 1) k<1><<<148, warps * 32>>>(out, iters, cyc);
      if (v == 2) k<2><<<148, warps * 32>>>(out, iters, cyc);
      if (v == 3) k<3><<<148, warps * 32>>>(out, iters, cyc);
      if (v == 4) k<4><<<148, warps * 32>>>(out, iters, cyc);
      if (v == 5) k<5><<<148, warps * 32>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-24s warps/SM %d: %6.0f cycles per 128-exp pass per warp (floor %d)\n", names[v], warps,
             double(h) / iters / (warps / 4), 1024);
    }
  return 0;
}
