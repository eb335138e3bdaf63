// attn_simt.cu -- causal softmax attention, forward and backward, SIMT fp32 arithmetic.
// Used by the fp32 parity path (and as the GPU reference for the tcgen05 kernels).
//   S = c·q kᵀ (c = 1/√d_h), −∞ above the diagonal, P = softmax, o = P v
//   dv = Pᵀ do ; dP = do vᵀ ; δ = rowsum(do⊙o) ; dS = P⊙(dP − δ) ; dq = c dS k ; dk = c dSᵀ q
// Layout: qkv [B·S, 3H] = [q | k | v] column blocks, head h at columns h·d_h; o / do [B·S, H];
// lse fp32 [B][n_h][S] (natural log); dqkv like qkv.
#include "common.cuh"

namespace tp {
namespace {

constexpr int NT = 128;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ float blk_sum(float v, float* red) {
  v = warp_sum(v);
  __syncthreads();
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  return t;
}
__device__ float blk_max(float v, float* red) {
  v = warp_max(v);
  __syncthreads();
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int i = 0; i < NT / 32; ++i) t = fmaxf(t, red[i]);
  return t;
}

template <typename T>
__global__ void __launch_bounds__(NT) fwd_kernel(int S, int nh, int dh, const T* __restrict__ qkv, T* __restrict__ o,
                                                 float* __restrict__ lse) {
  extern __shared__ float sm[];
  float* q = sm;        // [dh]
  float* sc = sm + dh;  // [S]
  __shared__ float red[NT / 32];
  const int i = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int H = nh * dh;
  const int64_t ld = 3ll * H;
  const int64_t row0 = static_cast<int64_t>(b) * S;
  const float c = rsqrtf(static_cast<float>(dh));
  for (int d = threadIdx.x; d < dh; d += NT) q[d] = to_f(qkv[(row0 + i) * ld + h * dh + d]);
  __syncthreads();
  float mx = -INFINITY;
  for (int j = threadIdx.x; j <= i; j += NT) {
    const T* kr = qkv + (row0 + j) * ld + H + h * dh;
    float s = 0.f;
    for (int d = 0; d < dh; ++d) s = fmaf(q[d], to_f(kr[d]), s);
    s *= c;
    sc[j] = s;
    mx = fmaxf(mx, s);
  }
  mx = blk_max(mx, red);
  float l = 0.f;
  for (int j = threadIdx.x; j <= i; j += NT) {
    const float e = __expf(sc[j] - mx);
    sc[j] = e;
    l += e;
  }
  l = blk_sum(l, red);
  if (threadIdx.x == 0) lse[(static_cast<int64_t>(b) * nh + h) * S + i] = mx + __logf(l);
  __syncthreads();
  const float inv = 1.f / l;
  for (int d = threadIdx.x; d < dh; d += NT) {
    float acc = 0.f;
    for (int j = 0; j <= i; ++j) acc = fmaf(sc[j], to_f(qkv[(row0 + j) * ld + 2 * H + h * dh + d]), acc);
    o[(row0 + i) * H + h * dh + d] = from_f<T>(acc * inv);
  }
}

// δ_i = Σ_d do_id · o_id, one warp per (row, head)
template <typename T>
__global__ void delta_kernel(int64_t rows, int S, int nh, int dh, const T* __restrict__ o, const T* __restrict__ dout,
                             float* __restrict__ delta) {
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= rows * nh) return;
  const int64_t row = w / nh;
  const int h = static_cast<int>(w % nh);
  const int H = nh * dh;
  float acc = 0.f;
  for (int d = lane; d < dh; d += 32) acc += to_f(o[row * H + h * dh + d]) * to_f(dout[row * H + h * dh + d]);
  acc = warp_sum(acc);
  if (lane == 0) {
    const int64_t b = row / S, p = row % S;
    delta[(b * nh + h) * S + p] = acc;
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) dq_kernel(int S, int nh, int dh, const T* __restrict__ qkv,
                                                const float* __restrict__ lse, const T* __restrict__ dout,
                                                const float* __restrict__ delta, T* __restrict__ dqkv) {
  extern __shared__ float sm[];
  float* q = sm;
  float* dov = sm + dh;
  float* ds = sm + 2 * dh;  // [S]
  const int i = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int H = nh * dh;
  const int64_t ld = 3ll * H;
  const int64_t row0 = static_cast<int64_t>(b) * S;
  const float c = rsqrtf(static_cast<float>(dh));
  for (int d = threadIdx.x; d < dh; d += NT) {
    q[d] = to_f(qkv[(row0 + i) * ld + h * dh + d]);
    dov[d] = to_f(dout[(row0 + i) * H + h * dh + d]);
  }
  __syncthreads();
  const float li = lse[(static_cast<int64_t>(b) * nh + h) * S + i];
  const float di = delta[(static_cast<int64_t>(b) * nh + h) * S + i];
  for (int j = threadIdx.x; j <= i; j += NT) {
    const T* kr = qkv + (row0 + j) * ld + H + h * dh;
    const T* vr = qkv + (row0 + j) * ld + 2 * H + h * dh;
    float s = 0.f, dp = 0.f;
    for (int d = 0; d < dh; ++d) {
      s = fmaf(q[d], to_f(kr[d]), s);
      dp = fmaf(dov[d], to_f(vr[d]), dp);
    }
    const float p = __expf(s * c - li);
    ds[j] = p * (dp - di);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < dh; d += NT) {
    float acc = 0.f;
    for (int j = 0; j <= i; ++j) acc = fmaf(ds[j], to_f(qkv[(row0 + j) * ld + H + h * dh + d]), acc);
    dqkv[(row0 + i) * ld + h * dh + d] = from_f<T>(acc * c);
  }
}

constexpr int CH = 2048;  // query rows per chunk in dk/dv

template <typename T>
__global__ void __launch_bounds__(NT) dkv_kernel(int S, int nh, int dh, const T* __restrict__ qkv,
                                                 const float* __restrict__ lse, const T* __restrict__ dout,
                                                 const float* __restrict__ delta, T* __restrict__ dqkv) {
  extern __shared__ float sm[];
  float* kk = sm;
  float* vv = sm + dh;
  float* P = sm + 2 * dh;        // [CH]
  float* dS = sm + 2 * dh + CH;  // [CH]
  const int j = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int H = nh * dh;
  const int64_t ld = 3ll * H;
  const int64_t row0 = static_cast<int64_t>(b) * S;
  const float c = rsqrtf(static_cast<float>(dh));
  for (int d = threadIdx.x; d < dh; d += NT) {
    kk[d] = to_f(qkv[(row0 + j) * ld + H + h * dh + d]);
    vv[d] = to_f(qkv[(row0 + j) * ld + 2 * H + h * dh + d]);
  }
  float dv_acc[2] = {0.f, 0.f}, dk_acc[2] = {0.f, 0.f};  // d = tid, tid + NT  (dh <= 256)
  for (int i0 = j; i0 < S; i0 += CH) {
    const int i1 = min(S, i0 + CH);
    __syncthreads();
    for (int i = i0 + threadIdx.x; i < i1; i += NT) {
      const T* qr = qkv + (row0 + i) * ld + h * dh;
      const T* dr = dout + (row0 + i) * H + h * dh;
      float s = 0.f, dp = 0.f;
      for (int d = 0; d < dh; ++d) {
        s = fmaf(to_f(qr[d]), kk[d], s);
        dp = fmaf(to_f(dr[d]), vv[d], dp);
      }
      const int64_t li = (static_cast<int64_t>(b) * nh + h) * S + i;
      const float p = __expf(s * c - lse[li]);
      P[i - i0] = p;
      dS[i - i0] = p * (dp - delta[li]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int d = threadIdx.x + u * NT;
      if (d >= dh) continue;
      float av = dv_acc[u], ak = dk_acc[u];
      for (int i = i0; i < i1; ++i) {
        av = fmaf(P[i - i0], to_f(dout[(row0 + i) * H + h * dh + d]), av);
        ak = fmaf(dS[i - i0], to_f(qkv[(row0 + i) * ld + h * dh + d]), ak);
      }
      dv_acc[u] = av;
      dk_acc[u] = ak;
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int d = threadIdx.x + u * NT;
    if (d >= dh) continue;
    dqkv[(row0 + j) * ld + H + h * dh + d] = from_f<T>(dk_acc[u] * c);
    dqkv[(row0 + j) * ld + 2 * H + h * dh + d] = from_f<T>(dv_acc[u]);
  }
}

template <typename K>
void set_smem(K k, size_t bytes) {
  if (bytes > 48 * 1024) TP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

template <typename T>
void attention_fwd_simt(int B, int S, int nh, int dh, const T* qkv, T* o, float* lse, cudaStream_t s) {
  TP_CHECK(dh <= 256 && S <= 50000, TAWPIPE_ECONFIG, "SIMT attention: d_h <= 256, S <= 50000");
  const size_t smem = (static_cast<size_t>(dh) + S) * sizeof(float);
  set_smem(fwd_kernel<T>, smem);
  fwd_kernel<T><<<dim3(S, nh, B), NT, smem, s>>>(S, nh, dh, qkv, o, lse);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
}

template <typename T>
void attention_bwd_simt(int B, int S, int nh, int dh, const T* qkv, const T* o, const float* lse, const T* dout,
                        T* dqkv, float* delta, cudaStream_t s) {
  TP_CHECK(dh <= 256 && S <= 50000, TAWPIPE_ECONFIG, "SIMT attention: d_h <= 256, S <= 50000");
  const int64_t rows = static_cast<int64_t>(B) * S;
  const int64_t warps = rows * nh;
  delta_kernel<T><<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, s>>>(rows, S, nh, dh, o, dout, delta);
  const size_t smem_q = (2 * static_cast<size_t>(dh) + S) * sizeof(float);
  set_smem(dq_kernel<T>, smem_q);
  dq_kernel<T><<<dim3(S, nh, B), NT, smem_q, s>>>(S, nh, dh, qkv, lse, dout, delta, dqkv);
  const size_t smem_kv = (2 * static_cast<size_t>(dh) + 2 * CH) * sizeof(float);
  set_smem(dkv_kernel<T>, smem_kv);
  dkv_kernel<T><<<dim3(S, nh, B), NT, smem_kv, s>>>(S, nh, dh, qkv, lse, dout, delta, dqkv);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches += 3;
}

template void attention_fwd_simt<float>(int, int, int, int, const float*, float*, float*, cudaStream_t);
template void attention_fwd_simt<bf16>(int, int, int, int, const bf16*, bf16*, float*, cudaStream_t);
template void attention_bwd_simt<float>(int, int, int, int, const float*, const float*, const float*, const float*,
                                        float*, float*, cudaStream_t);
template void attention_bwd_simt<bf16>(int, int, int, int, const bf16*, const bf16*, const float*, const bf16*, bf16*,
                                       float*, cudaStream_t);

}  // namespace tp
