// common.cuh -- shared declarations of libtawpipe's CUDA sources.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tawpipe.h"

namespace tp {

using bf16 = __nv_bfloat16;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TP_CUDA(x)                                                                                        \
  do {                                                                                                    \
    cudaError_t e_ = (x);                                                                                 \
    if (e_ != cudaSuccess)                                                                                \
      throw ::tp::Error(TAWPIPE_ERUNTIME, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " +       \
                                              __FILE__ + ":" + std::to_string(__LINE__) + " (" #x ")"); \
  } while (0)

#define TP_CHECK(cond, code, msg)                       \
  do {                                                  \
    if (!(cond)) throw ::tp::Error((code), (msg));      \
  } while (0)

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// ---------------------------------------------------------------- launch accounting
struct KernelStats {
  long launches = 0;
};
extern KernelStats g_kstats;

// ---------------------------------------------------------------- GEMM (gemm_tc.cu / gemm_simt.cu)
// RoPE in the bf16 epilogue of the QKV projection: output columns [0, cols) (q | k) are rotated per d_h-wide head;
// cs = [S][d_h] fp32 with cos(p·θ_i) in [0, d_h/2) and sin in [d_h/2, d_h); cs == nullptr: no RoPE
struct RopeEpi {
  const float* cs = nullptr;
  int S = 0, dh = 0;
  int64_t cols = 0;
};
struct GemmArgs {
  int64_t M, N, K;
  const void* A;
  int64_t lda;
  bool a_kmajor;
  const void* B;
  int64_t ldb;
  bool b_kmajor;
  void* C;
  int64_t ldc;
  bool c_f32;
  bool accumulate;
  const void* R;  // residual (same dtype / ld as C), nullable
  int epi = 0;     // 0 plain, 3 SwiGLU forward (C = gu or null, aux = y), 4 SwiGLU backward (C = dgu, aux = gu)
  void* aux = nullptr;
  int64_t ldx = 0;
  int64_t I = 0;
  RopeEpi rope{};
};
void gemm_tc_bf16(const GemmArgs& g, cudaStream_t s);   // tcgen05 + TMA + TMEM
template <typename T>
void gemm_simt(const GemmArgs& g, cudaStream_t s);      // generic strided SIMT (fp32 parity path)

// ---------------------------------------------------------------- attention (attn_*.cu)
template <typename T>
void attention_fwd_simt(int B, int S, int nh, int dh, const T* qkv, T* o, float* lse, cudaStream_t s);
template <typename T>
void attention_bwd_simt(int B, int S, int nh, int dh, const T* qkv, const T* o, const float* lse, const T* dout,
                        T* dqkv, float* delta, cudaStream_t s);
void attention_fwd_tc(int B, int S, int nh, int dh, const bf16* qkv, bf16* o, float* lse, cudaStream_t s);
// scratch: 2·B·n_h·S floats (δ and the log2-domain LSE); dq_acc: B·S·H floats.  With RoPE tables ([S][d_h/2] fp32,
// nullable) dq and dk are also rotated back by −p·θ (the inverse RoPE fused into the dq conversion and the dK epilogue)
void attention_bwd_tc(int B, int S, int nh, int dh, const bf16* qkv, const bf16* o, const float* lse,
                      const bf16* dout, bf16* dqkv, float* scratch, float* dq_acc, cudaStream_t s,
                      const float* rope_cos = nullptr, const float* rope_sin = nullptr);
bool attention_tc_supported(int S, int dh);

// ---------------------------------------------------------------- elementwise / norm / loss / optimizer
template <typename T>
void embed_fwd(const int32_t* tok, int64_t tok_stride_seq, int B, int S, const T* E, int H, T* h, cudaStream_t s);
// Deterministic embedding backward (embed.cu): dE[v] += Σ_{p : tok[p] = v} dh[p], the positions of each token summed
// in ascending order in fp32 (a stable radix sort of (token, position) pairs, then one segment per token), so the
// result is bit-reproducible run to run.  scratch: embed_bwd_scratch_bytes(B·S) bytes, device.
size_t embed_bwd_scratch_bytes(int64_t T);
void embed_bwd(const int32_t* tok, int64_t tok_stride_seq, int B, int S, const void* dh, bool dh_f32, int H, int V,
               float* dE, void* scratch, size_t scratch_bytes, cudaStream_t s);
template <typename T>
void rmsnorm_fwd(const T* x, const T* g, T* y, float* rstd, int64_t rows, int H, float eps, cudaStream_t s);
// dx = (res ? res : 0) + RMSNorm'(dy); dg_acc += Σ_rows dy⊙x⊙r (fp32).  The row-block partial sums of dγ go to
// dg_scratch (≥ rmsnorm_bwd_scratch_floats(rows, H) floats) and are added in block order: deterministic
size_t rmsnorm_bwd_scratch_floats(int64_t rows, int H);
template <typename T>
void rmsnorm_bwd(const T* dy, const T* x, const T* g, const float* rstd, const T* res, T* dx, float* dg_acc,
                 float* dg_scratch, int64_t rows, int H, cudaStream_t s);
template <typename T>
void rope_apply(T* qkv, int B, int S, int nh, int dh, const float* cos, const float* sin, bool inverse, int ncols_blocks,
                cudaStream_t s);
template <typename T>
void swiglu_fwd(const T* gu, T* y, int64_t rows, int I, cudaStream_t s);
template <typename T>
void swiglu_bwd(const T* dy, const T* gu, T* dgu, int64_t rows, int I, cudaStream_t s);
// logits [rows, V] in place -> dz; loss_rows[r] = LSE - z[t]
template <typename T>
void cross_entropy(T* logits, const int32_t* targets, int64_t rows, int V, float inv_denom, float* loss_rows,
                   cudaStream_t s);
void sum_f32_to_f64(const float* x, int64_t n, double* out_accum, cudaStream_t s);
template <typename T>
void cast_f32(const float* x, T* y, int64_t n, cudaStream_t s);
template <typename T>
void cast_to_f32(const T* x, float* y, int64_t n, cudaStream_t s);
// y = (T)(a + b) with a in T and b fp32 (one hop of the ring gradient reduction)
template <typename T>
void add_cast(const T* a, const float* b, T* y, int64_t n, cudaStream_t s);
template <typename T>
void init_normal(T* wire, float* master, int64_t n, int64_t global_off, uint64_t seed, float std, cudaStream_t s);
void fill_f32(float* x, int64_t n, float v, cudaStream_t s);
// emulated link time: one thread spins on the global timer for `seconds` on stream s (NEXT-3)
void link_delay(double seconds, cudaStream_t s);

struct AdamParams {
  float lr, beta1, beta2, eps, wd;
  float bc1, bc2;  // 1 - beta^t
};
struct AdamRanges {  // no-decay ranges [lo, hi) in unit coordinates (RMSNorm gains, R1); empty ranges: lo = hi = 0
  int64_t lo[2] = {0, 0}, hi[2] = {0, 0};
};
// Gradient sources of one owned stripe, grouped: group gi holds sources [group_end[gi−1], group_end[gi]) (member
// order); bit si of f32_mask: source si is fp32, else the wire dtype.  Pointers may be peer (IPC-mapped) memory.
struct GradSources {
  const void* p[16] = {};
  int n_groups = 0;
  int group_end[8] = {};
  unsigned f32_mask = 0;
};
// g = Σ_groups Σ_members (fp32), then AdamW on master / m / v [n] and wire[n] = W(master) (a9)
template <typename W>
void adamw_grouped(const GradSources& src, float* master, float* m, float* v, W* wire, int64_t n, int64_t unit_off,
                   const AdamRanges& nd, const AdamParams& p, cudaStream_t s);

// cos / sin of p·θ_i, θ_i = theta^(−2i/d_h), i < d_h/2, p < S: computed in fp64, stored fp32 (R10, R13); [S][d_h/2]
void rope_tables_host(int S, int dh, double theta, std::vector<float>& cos_t, std::vector<float>& sin_t);

// ---------------------------------------------------------------- errors at the C ABI
void set_last_error(const std::string& msg);
template <typename F>
int guarded(F f) {
  try {
    f();
    return TAWPIPE_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TAWPIPE_ERUNTIME;
  }
}

}  // namespace tp
