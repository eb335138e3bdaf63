// embed.cu -- deterministic embedding backward (a4): dE[v] += Σ_{p : x_p = v} dh_p (SURVEY.md §8(c) step 1 backward,
// "dE[x_p] += dh0[p]"; reading: token-sorted on the GPU).
//
// The positions of one micro-batch are sorted by token with a stable radix sort (library primitive: CUB), so each
// token's positions form one contiguous segment in ascending position order; one CTA per segment sums its rows in
// that order in fp32 and adds the sum into the fp32 accumulator row.  Every row of dE is written by exactly one CTA
// per launch and micro-batches are applied in stream order, so the result is bit-identical run to run (the
// atomicAdd scatter of round 1 was not).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "common.cuh"

namespace tp {
namespace {

__global__ void embed_keys_kernel(const int32_t* __restrict__ tok, int64_t stride_seq, int S, int64_t T,
                                  int32_t* __restrict__ keys, int32_t* __restrict__ pos) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < T;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = p / S, s = p % S;
    keys[p] = tok[b * stride_seq + s];
    pos[p] = static_cast<int32_t>(p);
  }
}

// one CTA per sorted index i; the CTA whose i starts a segment (first index or a new token) owns that token
template <typename T>
__global__ void __launch_bounds__(256) embed_segment_kernel(const int32_t* __restrict__ keys,
                                                            const int32_t* __restrict__ pos, int64_t n,
                                                            const T* __restrict__ dh, int H, float* __restrict__ dE) {
  const int64_t i = blockIdx.x;
  const int32_t v = keys[i];
  if (i > 0 && keys[i - 1] == v) return;
  int64_t end = i + 1;
  while (end < n && keys[end] == v) ++end;
  float* row = dE + static_cast<int64_t>(v) * H;
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    float acc = 0.f;
    for (int64_t j = i; j < end; ++j) acc += to_f(dh[static_cast<int64_t>(pos[j]) * H + c]);   // ascending position
    row[c] += acc;
  }
}

// bf16 rows, 8 columns per thread (H % 8 == 0)
__global__ void __launch_bounds__(256) embed_segment_v8_kernel(const int32_t* __restrict__ keys,
                                                               const int32_t* __restrict__ pos, int64_t n,
                                                               const bf16* __restrict__ dh, int H,
                                                               float* __restrict__ dE) {
  const int64_t i = blockIdx.x;
  const int32_t v = keys[i];
  if (i > 0 && keys[i - 1] == v) return;
  int64_t end = i + 1;
  while (end < n && keys[end] == v) ++end;
  float* row = dE + static_cast<int64_t>(v) * H;
  for (int c = threadIdx.x * 8; c < H; c += blockDim.x * 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int64_t j = i; j < end; ++j) {
      const uint4 u = *reinterpret_cast<const uint4*>(dh + static_cast<int64_t>(pos[j]) * H + c);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h2[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
    float4* r4 = reinterpret_cast<float4*>(row + c);
    float4 a = r4[0], b = r4[1];
    a.x += acc[0]; a.y += acc[1]; a.z += acc[2]; a.w += acc[3];
    b.x += acc[4]; b.y += acc[5]; b.z += acc[6]; b.w += acc[7];
    r4[0] = a;
    r4[1] = b;
  }
}

size_t cub_bytes(int64_t T) {
  size_t bytes = 0;
  TP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const int32_t*>(nullptr),
                                          static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                          static_cast<int32_t*>(nullptr), static_cast<int>(T)));
  return bytes;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t embed_bwd_scratch_bytes(int64_t T) { return 4 * align256(static_cast<size_t>(T) * 4) + align256(cub_bytes(T)); }

void embed_bwd(const int32_t* tok, int64_t stride_seq, int B, int S, const void* dh, bool dh_f32, int H, int V,
               float* dE, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const int64_t T = static_cast<int64_t>(B) * S;
  TP_CHECK(T >= 1 && T < (1ll << 31), TAWPIPE_ECONFIG, "embedding backward: 1 <= B·S < 2^31");
  TP_CHECK(scratch != nullptr && scratch_bytes >= embed_bwd_scratch_bytes(T), TAWPIPE_ECONFIG,
           "embedding backward: scratch too small");
  char* p = static_cast<char*>(scratch);
  const size_t a = align256(static_cast<size_t>(T) * 4);
  int32_t* keys_in = reinterpret_cast<int32_t*>(p);
  int32_t* keys_out = reinterpret_cast<int32_t*>(p + a);
  int32_t* pos_in = reinterpret_cast<int32_t*>(p + 2 * a);
  int32_t* pos_out = reinterpret_cast<int32_t*>(p + 3 * a);
  void* temp = p + 4 * a;
  size_t temp_bytes = scratch_bytes - 4 * a;
  embed_keys_kernel<<<static_cast<unsigned>(std::min<int64_t>((T + 255) / 256, 148 * 16)), 256, 0, s>>>(
      tok, stride_seq, S, T, keys_in, pos_in);
  TP_CUDA(cudaGetLastError());
  int end_bit = 1;
  while (end_bit < 31 && (1ll << end_bit) < V) ++end_bit;
  TP_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, pos_in, pos_out, static_cast<int>(T), 0,
                                          end_bit, s));
  if (!dh_f32 && H % 8 == 0)
    embed_segment_v8_kernel<<<static_cast<unsigned>(T), 256, 0, s>>>(keys_out, pos_out, T,
                                                                      static_cast<const bf16*>(dh), H, dE);
  else if (dh_f32)
    embed_segment_kernel<float><<<static_cast<unsigned>(T), 256, 0, s>>>(keys_out, pos_out, T,
                                                                         static_cast<const float*>(dh), H, dE);
  else
    embed_segment_kernel<bf16><<<static_cast<unsigned>(T), 256, 0, s>>>(keys_out, pos_out, T,
                                                                        static_cast<const bf16*>(dh), H, dE);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches += 2;   // this library's kernels: keys, segments (the radix sort is CUB's)
}

}  // namespace tp
