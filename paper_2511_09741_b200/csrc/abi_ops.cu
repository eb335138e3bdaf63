// abi_ops.cu -- kernel-level C ABI entries (include/tawpipe.h, "kernel-level entry points"): each runs exactly the
// kernel(s) the training step launches for that operation, on caller-owned device buffers, so the per-op parity
// tests (tests/test_gpu_ops.py, tests/test_gpu_kernels.py) check the very code the bench times against the oracle's
// per-op functions.  No context is needed (no tawpipe_bootstrap); the caller's current device is used.
#include <cuda.h>

#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "peer.cuh"

using namespace tp;

namespace {

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

void check_dtype(int dtype) {
  TP_CHECK(dtype == TAWPIPE_FP32 || dtype == TAWPIPE_BF16, TAWPIPE_ECONFIG, "dtype must be TAWPIPE_FP32 or TAWPIPE_BF16");
}

bool env_is(const char* name, const char* val) {
  const char* e = std::getenv(name);
  return e && std::string(e) == val;
}

}  // namespace

extern "C" {

int tawpipe_gemm(int dtype, int64_t M, int64_t N, int64_t K, const void* A, int64_t a_ld, int a_kmajor, const void* B,
                 int64_t b_ld, int b_kmajor, void* C, int64_t c_ld, int c_f32, int accumulate, const void* R,
                 void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    GemmArgs a{M, N, K, A, a_ld, a_kmajor != 0, B, b_ld, b_kmajor != 0, C, c_ld, c_f32 != 0, accumulate != 0, R};
    if (dtype == TAWPIPE_BF16) {
      if (env_is("TAWPIPE_GEMM", "simt"))
        gemm_simt<bf16>(a, as_stream(stream));
      else
        gemm_tc_bf16(a, as_stream(stream));
    } else {
      gemm_simt<float>(a, as_stream(stream));
    }
  });
}

int tawpipe_gemm_rope(int64_t M, int64_t N, int64_t K, const void* x, const void* w, void* qkv, int S, int d_h,
                      float theta, int64_t rope_cols, void* stream) {
  return guarded([&] {
    TP_CHECK(S >= 1 && d_h >= 64 && d_h % 64 == 0, TAWPIPE_ECONFIG, "gemm_rope: S >= 1, d_h % 64 == 0");
    cudaStream_t s = as_stream(stream);
    std::vector<float> cs, sn;
    rope_tables_host(S, d_h, theta, cs, sn);
    const int half = d_h / 2;
    std::vector<float> both(static_cast<size_t>(S) * d_h);
    for (int p = 0; p < S; ++p)
      for (int i = 0; i < half; ++i) {
        both[static_cast<size_t>(p) * d_h + i] = cs[static_cast<size_t>(p) * half + i];
        both[static_cast<size_t>(p) * d_h + half + i] = sn[static_cast<size_t>(p) * half + i];
      }
    float* d = nullptr;
    TP_CUDA(cudaMallocAsync(&d, both.size() * 4, s));
    TP_CUDA(cudaMemcpyAsync(d, both.data(), both.size() * 4, cudaMemcpyHostToDevice, s));
    GemmArgs a{M, N, K, x, K, true, w, K, true, qkv, N, false, false, nullptr};
    a.rope.cs = d;
    a.rope.S = S;
    a.rope.dh = d_h;
    a.rope.cols = rope_cols;
    gemm_tc_bf16(a, s);
    TP_CUDA(cudaFreeAsync(d, s));
    TP_CUDA(cudaStreamSynchronize(s));
  });
}

int tawpipe_gemm_swiglu(int64_t M, int64_t I, int64_t K, const void* x, const void* w_gu, void* gu, void* y,
                        void* stream) {
  return guarded([&] {
    TP_CHECK(y != nullptr, TAWPIPE_ECONFIG, "y is NULL");
    GemmArgs a{M, 2 * I, K, x, K, true, w_gu, K, true, gu, 2 * I, false, false, nullptr};
    a.epi = 3;
    a.aux = y;
    a.ldx = I;
    a.I = I;
    gemm_tc_bf16(a, as_stream(stream));
  });
}

int tawpipe_gemm_swiglu_bwd(int64_t M, int64_t I, int64_t K, const void* dh, const void* w_down, const void* gu,
                            void* dgu, void* stream) {
  return guarded([&] {
    GemmArgs a{M, I, K, dh, K, true, w_down, I, false, dgu, 2 * I, false, false, nullptr};
    a.epi = 4;
    a.aux = const_cast<void*>(gu);
    a.ldx = 2 * I;
    a.I = I;
    gemm_tc_bf16(a, as_stream(stream));
  });
}

int tawpipe_attention_fwd(int dtype, int B, int S, int n_h, int d_h, const void* qkv, void* o, float* lse,
                          void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    cudaStream_t s = as_stream(stream);
    if (dtype == TAWPIPE_FP32)
      attention_fwd_simt<float>(B, S, n_h, d_h, (const float*)qkv, (float*)o, lse, s);
    else if (attention_tc_supported(S, d_h) && !env_is("TAWPIPE_ATTN", "simt"))
      attention_fwd_tc(B, S, n_h, d_h, (const bf16*)qkv, (bf16*)o, lse, s);
    else
      attention_fwd_simt<bf16>(B, S, n_h, d_h, (const bf16*)qkv, (bf16*)o, lse, s);
  });
}

int tawpipe_attention_bwd(int dtype, int B, int S, int n_h, int d_h, const void* qkv, const void* o, const float* lse,
                          const void* do_, void* dqkv, float* scratch, float* dq_acc, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    cudaStream_t s = as_stream(stream);
    if (dtype == TAWPIPE_FP32)
      attention_bwd_simt<float>(B, S, n_h, d_h, (const float*)qkv, (const float*)o, lse, (const float*)do_,
                                (float*)dqkv, scratch, s);
    else if (attention_tc_supported(S, d_h) && !env_is("TAWPIPE_ATTN", "simt"))
      attention_bwd_tc(B, S, n_h, d_h, (const bf16*)qkv, (const bf16*)o, lse, (const bf16*)do_, (bf16*)dqkv, scratch,
                       dq_acc, s);
    else
      attention_bwd_simt<bf16>(B, S, n_h, d_h, (const bf16*)qkv, (const bf16*)o, lse, (const bf16*)do_, (bf16*)dqkv,
                               scratch, s);
  });
}

int tawpipe_attention_bwd_rope(int dtype, int B, int S, int n_h, int d_h, float theta, const void* qkv, const void* o,
                               const float* lse, const void* do_, void* dqkv, float* scratch, float* dq_acc,
                               void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    cudaStream_t s = as_stream(stream);
    std::vector<float> cs, sn;
    rope_tables_host(S, d_h, theta, cs, sn);
    float *dc = nullptr, *dsn = nullptr;
    TP_CUDA(cudaMallocAsync(&dc, cs.size() * 4, s));
    TP_CUDA(cudaMallocAsync(&dsn, sn.size() * 4, s));
    TP_CUDA(cudaMemcpyAsync(dc, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, s));
    TP_CUDA(cudaMemcpyAsync(dsn, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice, s));
    if (dtype == TAWPIPE_BF16 && attention_tc_supported(S, d_h) && !env_is("TAWPIPE_ATTN", "simt")) {
      attention_bwd_tc(B, S, n_h, d_h, (const bf16*)qkv, (const bf16*)o, lse, (const bf16*)do_, (bf16*)dqkv, scratch,
                       dq_acc, s, dc, dsn);
    } else if (dtype == TAWPIPE_BF16) {
      attention_bwd_simt<bf16>(B, S, n_h, d_h, (const bf16*)qkv, (const bf16*)o, lse, (const bf16*)do_, (bf16*)dqkv,
                               scratch, s);
      rope_apply<bf16>((bf16*)dqkv, B, S, n_h, d_h, dc, dsn, true, 2, s);
    } else {
      attention_bwd_simt<float>(B, S, n_h, d_h, (const float*)qkv, (const float*)o, lse, (const float*)do_,
                                (float*)dqkv, scratch, s);
      rope_apply<float>((float*)dqkv, B, S, n_h, d_h, dc, dsn, true, 2, s);
    }
    TP_CUDA(cudaFreeAsync(dc, s));
    TP_CUDA(cudaFreeAsync(dsn, s));
    TP_CUDA(cudaStreamSynchronize(s));
  });
}

int tawpipe_rmsnorm_fwd(int dtype, int64_t rows, int H, const void* x, const void* gamma, float eps, void* y,
                        float* rstd, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (dtype == TAWPIPE_BF16)
      rmsnorm_fwd<bf16>((const bf16*)x, (const bf16*)gamma, (bf16*)y, rstd, rows, H, eps, as_stream(stream));
    else
      rmsnorm_fwd<float>((const float*)x, (const float*)gamma, (float*)y, rstd, rows, H, eps, as_stream(stream));
  });
}

int tawpipe_rmsnorm_bwd(int dtype, int64_t rows, int H, const void* dy, const void* x, const void* gamma,
                        const float* rstd, const void* res, void* dx, float* dgamma_acc, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    cudaStream_t s = as_stream(stream);
    float* scratch = nullptr;   // dγ row-block partials, stream-ordered allocation for this call
    TP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), rmsnorm_bwd_scratch_floats(rows, H) * 4, s));
    if (dtype == TAWPIPE_BF16)
      rmsnorm_bwd<bf16>((const bf16*)dy, (const bf16*)x, (const bf16*)gamma, rstd, (const bf16*)res, (bf16*)dx,
                        dgamma_acc, scratch, rows, H, s);
    else
      rmsnorm_bwd<float>((const float*)dy, (const float*)x, (const float*)gamma, rstd, (const float*)res, (float*)dx,
                         dgamma_acc, scratch, rows, H, s);
    TP_CUDA(cudaFreeAsync(scratch, s));
  });
}

int tawpipe_rope(int dtype, int B, int S, int n_h, int d_h, float theta, void* qkv, int inverse, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    TP_CHECK(B >= 1 && S >= 1 && n_h >= 1 && d_h >= 2 && d_h % 2 == 0, TAWPIPE_ECONFIG, "rope: bad shape");
    cudaStream_t s = as_stream(stream);
    std::vector<float> cs, sn;
    rope_tables_host(S, d_h, theta, cs, sn);
    float *dc = nullptr, *dsn = nullptr;
    TP_CUDA(cudaMallocAsync(&dc, cs.size() * 4, s));
    TP_CUDA(cudaMallocAsync(&dsn, sn.size() * 4, s));
    TP_CUDA(cudaMemcpyAsync(dc, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, s));
    TP_CUDA(cudaMemcpyAsync(dsn, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice, s));
    if (dtype == TAWPIPE_BF16)
      rope_apply<bf16>((bf16*)qkv, B, S, n_h, d_h, dc, dsn, inverse != 0, 2, s);
    else
      rope_apply<float>((float*)qkv, B, S, n_h, d_h, dc, dsn, inverse != 0, 2, s);
    TP_CUDA(cudaFreeAsync(dc, s));
    TP_CUDA(cudaFreeAsync(dsn, s));
    TP_CUDA(cudaStreamSynchronize(s));   // the pageable host tables go out of scope
  });
}

int tawpipe_swiglu_fwd(int dtype, int64_t rows, int I, const void* gu, void* y, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (dtype == TAWPIPE_BF16)
      swiglu_fwd<bf16>((const bf16*)gu, (bf16*)y, rows, I, as_stream(stream));
    else
      swiglu_fwd<float>((const float*)gu, (float*)y, rows, I, as_stream(stream));
  });
}

int tawpipe_swiglu_bwd(int dtype, int64_t rows, int I, const void* dy, const void* gu, void* dgu, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (dtype == TAWPIPE_BF16)
      swiglu_bwd<bf16>((const bf16*)dy, (const bf16*)gu, (bf16*)dgu, rows, I, as_stream(stream));
    else
      swiglu_bwd<float>((const float*)dy, (const float*)gu, (float*)dgu, rows, I, as_stream(stream));
  });
}

int tawpipe_cross_entropy(int dtype, int64_t rows, int V, void* logits, const int32_t* targets, float inv_denom,
                          float* loss_rows, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (dtype == TAWPIPE_BF16)
      cross_entropy<bf16>((bf16*)logits, targets, rows, V, inv_denom, loss_rows, as_stream(stream));
    else
      cross_entropy<float>((float*)logits, targets, rows, V, inv_denom, loss_rows, as_stream(stream));
  });
}

int tawpipe_embed_fwd(int dtype, int B, int S, const int32_t* tokens, int64_t tok_stride, const void* E, int H, void* h,
                      void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    if (dtype == TAWPIPE_BF16)
      embed_fwd<bf16>(tokens, tok_stride, B, S, (const bf16*)E, H, (bf16*)h, as_stream(stream));
    else
      embed_fwd<float>(tokens, tok_stride, B, S, (const float*)E, H, (float*)h, as_stream(stream));
  });
}

int tawpipe_embed_bwd(int dtype, int B, int S, const int32_t* tokens, int64_t tok_stride, const void* dh, int H, int V,
                      float* dE, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    cudaStream_t s = as_stream(stream);
    const size_t bytes = embed_bwd_scratch_bytes(static_cast<int64_t>(B) * S);
    void* scratch = nullptr;
    TP_CUDA(cudaMallocAsync(&scratch, bytes, s));
    embed_bwd(tokens, tok_stride, B, S, dh, dtype == TAWPIPE_FP32, H, V, dE, scratch, bytes, s);
    TP_CUDA(cudaFreeAsync(scratch, s));
  });
}

int tawpipe_group_partial(int wire_dtype, int n_src, const float* const* srcs, int64_t n, void* out, void* stream) {
  return guarded([&] {
    check_dtype(wire_dtype);
    TP_CHECK(n_src >= 1 && n_src <= kMaxPartialSources && srcs && out && n >= 0, TAWPIPE_ECONFIG,
             "group_partial: 1..8 sources, non-NULL pointers, n >= 0");
    if (n == 0) return;
    PartialSources src;
    for (int i = 0; i < n_src; ++i) {
      TP_CHECK(srcs[i] && reinterpret_cast<uintptr_t>(srcs[i]) % 16 == 0, TAWPIPE_ECONFIG,
               "group_partial: sources must be 16-byte aligned");
      src.p[src.n++] = srcs[i];
    }
    TP_CHECK(reinterpret_cast<uintptr_t>(out) % 16 == 0, TAWPIPE_ECONFIG, "group_partial: out must be 16-byte aligned");
    if (wire_dtype == TAWPIPE_BF16)
      group_partial<bf16>(src, static_cast<bf16*>(out), n, as_stream(stream));
    else
      group_partial<float>(src, static_cast<float*>(out), n, as_stream(stream));
  });
}

int tawpipe_adamw(int wire_dtype, int n_groups, const int* group_sizes, const void* const* srcs, const int* src_is_f32,
                  float* master, float* m, float* v, void* wire, int64_t n, int64_t unit_off, const int64_t* no_decay,
                  const float* hyper, int step, void* stream) {
  return guarded([&] {
    check_dtype(wire_dtype);
    TP_CHECK(n_groups >= 1 && n_groups <= 8 && group_sizes && srcs && src_is_f32 && hyper && step >= 1,
             TAWPIPE_ECONFIG, "adamw: 1..8 groups, non-NULL sources / flags / hyper-parameters, step >= 1");
    GradSources src;
    src.n_groups = n_groups;
    int k = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
      TP_CHECK(group_sizes[gi] >= 1 && k + group_sizes[gi] <= 16, TAWPIPE_ECONFIG, "adamw: 1..16 sources in total");
      for (int i = 0; i < group_sizes[gi]; ++i, ++k) {
        src.p[k] = srcs[k];
        if (src_is_f32[k]) src.f32_mask |= 1u << k;
      }
      src.group_end[gi] = k;
    }
    AdamRanges nd;
    if (no_decay)
      for (int r = 0; r < 2; ++r) {
        nd.lo[r] = no_decay[2 * r];
        nd.hi[r] = no_decay[2 * r + 1];
      }
    AdamParams hp;
    hp.lr = hyper[0];
    hp.beta1 = hyper[1];
    hp.beta2 = hyper[2];
    hp.eps = hyper[3];
    hp.wd = hyper[4];
    hp.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(hyper[1]), step));
    hp.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(hyper[2]), step));
    if (wire_dtype == TAWPIPE_BF16)
      adamw_grouped<bf16>(src, master, m, v, (bf16*)wire, n, unit_off, nd, hp, as_stream(stream));
    else
      adamw_grouped<float>(src, master, m, v, (float*)wire, n, unit_off, nd, hp, as_stream(stream));
  });
}

}  // extern "C"
