// gemm_simt.cu -- generic strided SIMT GEMM (fp32 FMA, no tensor cores).
// The fp32 parity path (TAWPIPE_FP32) runs every contraction through this kernel: TF32 tensor cores
// would cost ~1e-3 relative error and break the 1e-5 loss tolerance (SURVEY.md §7 "hard parts" 3).
#include "common.cuh"

namespace tp {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

template <typename T, int EPI>  // EPI 0: store T (+R), 1: store f32, 2: accumulate f32
__global__ void __launch_bounds__(256) gemm_simt_kernel(int64_t M, int64_t N, int64_t K, const T* __restrict__ A,
                                                        int64_t sam, int64_t sak, const T* __restrict__ B, int64_t sbn,
                                                        int64_t sbk, void* __restrict__ C, int64_t ldc,
                                                        const T* __restrict__ R) {
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * TM, n0 = static_cast<int64_t>(blockIdx.x) * TN;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      int mm, kk;
      if (sak == 1) { kk = i % TK; mm = i / TK; } else { mm = i % TM; kk = i / TM; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? to_f(A[gm * sam + gk * sak]) : 0.f;
    }
    for (int i = threadIdx.x; i < TN * TK; i += 256) {
      int nn, kk;
      if (sbk == 1) { kk = i % TK; nn = i / TK; } else { nn = i % TN; kk = i / TN; }
      const int64_t gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < K) ? to_f(B[gn * sbn + gk * sbk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (EPI == 0) {
        if (R) v += to_f(R[gm * ldc + gn]);
        reinterpret_cast<T*>(C)[gm * ldc + gn] = from_f<T>(v);
      } else if (EPI == 1) {
        reinterpret_cast<float*>(C)[gm * ldc + gn] = v;
      } else {
        reinterpret_cast<float*>(C)[gm * ldc + gn] += v;
      }
    }
  }
}

}  // namespace

template <typename T>
void gemm_simt(const GemmArgs& g, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((g.N + TN - 1) / TN), static_cast<unsigned>((g.M + TM - 1) / TM));
  const int64_t sam = g.a_kmajor ? g.lda : 1, sak = g.a_kmajor ? 1 : g.lda;
  const int64_t sbn = g.b_kmajor ? g.ldb : 1, sbk = g.b_kmajor ? 1 : g.ldb;
  const T* A = static_cast<const T*>(g.A);
  const T* B = static_cast<const T*>(g.B);
  const T* R = static_cast<const T*>(g.R);
  if (!g.c_f32)
    gemm_simt_kernel<T, 0><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, sam, sak, B, sbn, sbk, g.C, g.ldc, R);
  else if (g.accumulate)
    gemm_simt_kernel<T, 2><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, sam, sak, B, sbn, sbk, g.C, g.ldc, R);
  else
    gemm_simt_kernel<T, 1><<<grid, 256, 0, s>>>(g.M, g.N, g.K, A, sam, sak, B, sbn, sbk, g.C, g.ldc, R);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
}

template void gemm_simt<float>(const GemmArgs&, cudaStream_t);
template void gemm_simt<bf16>(const GemmArgs&, cudaStream_t);

}  // namespace tp
