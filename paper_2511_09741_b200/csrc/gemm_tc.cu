// gemm_tc.cu -- persistent, warp-specialised tcgen05 GEMM for sm_100a (bf16 in, fp32 accumulate in TMEM).
//
//   C[M,N] (+)= Σ_k A(m,k) · B(n,k)      (+ R[M,N] residual)
//
// Used for every dense contraction of the decoder layer (QKV, O, gate/up, down,
// their dgrad and wgrad, and the LM head), which are the method's "dense contractions" (north_star).
//   forward  y  = x·Wᵀ   : A = x  (K-major), B = W  (K-major)
//   dgrad    dx = dy·W   : A = dy (K-major), B = W  (MN-major: contraction runs over W's rows)
//   wgrad    dW += dyᵀ·x : A = dy (MN-major), B = x (MN-major), C fp32 accumulate (grad accumulator)
//
// Roles (192 threads, one CTA per SM, persistent over output tiles; the producer and MMA warps take the highest
// warp ids of their SMSPs so that the hi-warp-id-first issue arbitration never starves them behind epilogue warps):
//   warp 4  TMA producer: 128×64 A tile + BN×64 B tile per stage, SWIZZLE_128B, mbarrier complete_tx
//   warp 5  MMA issuer:   one thread issues 4 × tcgen05.mma (M=128, N=BN, K=16) per stage into a TMEM
//                         accumulator; tcgen05.commit frees the smem stage / publishes the accumulator
//   warps 0-3 epilogue:   tcgen05.ld 32 columns at a time → fp32 → (+R / +=C) → bf16 or fp32 stores
// Two TMEM accumulators (2 × BN columns) let the epilogue of tile i overlap the mainloop of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <set>
#include <string>
#include <utility>

#include "common.cuh"
#include "ptx.cuh"

namespace tp {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;   // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;   // 32 / 16 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;
};

enum Epi : int { EPI_BF16 = 0, EPI_F32_STORE = 1, EPI_F32_ACC = 2, EPI_SWIGLU_FWD = 3, EPI_SWIGLU_BWD = 4 };

__device__ __forceinline__ float silu_sig(float u) { return 1.f / (1.f + __expf(-u)); }

// Epilogue of one output tile for this thread's accumulator row: TMEM columns [0, BN) of `tbase` hold
// C[row, nb·BN ..) (SwiGLU forward: gate u in [0, BN/2), up w in [BN/2, BN) of features nb·BN/2 ..).
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(uint32_t tbase, int64_t row, int nb, void* __restrict__ C, int64_t ldc,
                                              const bf16* __restrict__ R, void* __restrict__ aux, int64_t ldx,
                                              int64_t I, const RopeEpi& rope) {
  if (EPI == EPI_BF16 && rope.cs != nullptr && static_cast<int64_t>(nb) * BN < rope.cols) {
    // RoPE of the QKV projection in its epilogue (rotate-half, angle p·θ_i with p = row mod S): the tile holds whole
    // heads (BN and the head width divide each other's multiples: heads are d_h-aligned, tiles BN-aligned), so the
    // partner column i + d_h/2 of every column i is in the same tile; cos in cs[p][0, d_h/2), sin in [d_h/2, d_h)
    const int dh = rope.dh, half = dh / 2;
    const float* cs = rope.cs + (row % rope.S) * dh;
#pragma unroll 1
    for (int hb = 0; hb < BN; hb += dh) {
#pragma unroll 1
      for (int c = 0; c < half; c += 32) {
        uint32_t r1[32], r2[32];
        tmem_ld32(tbase + hb + c, r1);
        tmem_ld32(tbase + hb + half + c, r2);
        tmem_wait_ld();
        float y1[32], y2[32];
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 cc = reinterpret_cast<const float4*>(cs + c)[q4];
          const float4 ss = reinterpret_cast<const float4*>(cs + half + c)[q4];
          const float cv[4] = {cc.x, cc.y, cc.z, cc.w}, sv[4] = {ss.x, ss.y, ss.z, ss.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x1 = __uint_as_float(r1[4 * q4 + e]), x2 = __uint_as_float(r2[4 * q4 + e]);
            y1[4 * q4 + e] = x1 * cv[e] - x2 * sv[e];
            y2[4 * q4 + e] = x2 * cv[e] + x1 * sv[e];
          }
        }
        bf16* d1 = reinterpret_cast<bf16*>(C) + row * ldc + static_cast<int64_t>(nb) * BN + hb + c;
        bf16* d2 = d1 + half;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          reinterpret_cast<uint4*>(d1)[v] = make_uint4(pack_bf16(y1[8 * v], y1[8 * v + 1]), pack_bf16(y1[8 * v + 2], y1[8 * v + 3]),
                                                       pack_bf16(y1[8 * v + 4], y1[8 * v + 5]), pack_bf16(y1[8 * v + 6], y1[8 * v + 7]));
          reinterpret_cast<uint4*>(d2)[v] = make_uint4(pack_bf16(y2[8 * v], y2[8 * v + 1]), pack_bf16(y2[8 * v + 2], y2[8 * v + 3]),
                                                       pack_bf16(y2[8 * v + 4], y2[8 * v + 5]), pack_bf16(y2[8 * v + 6], y2[8 * v + 7]));
        }
      }
    }
    return;
  }
  if (EPI == EPI_SWIGLU_FWD) {
    // accumulator columns [0, BN/2) = gate u, [BN/2, BN) = up w of output features nb·BN/2 ..:
    // y = SiLU(u)·w -> aux [rows, I] ; optionally (C != nullptr) u, w -> C = gu [rows, 2I]
#pragma unroll 1
    for (int c = 0; c < BN / 2; c += 32) {
      uint32_t ru[32], rw[32];
      tmem_ld32(tbase + c, ru);
      tmem_ld32(tbase + BN / 2 + c, rw);
      tmem_wait_ld();
      const int64_t col = static_cast<int64_t>(nb) * (BN / 2) + c;
      uint4* y4 = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(aux) + row * ldx + col);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float yv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float u = __uint_as_float(ru[v * 8 + e]), w = __uint_as_float(rw[v * 8 + e]);
          yv[e] = u * silu_sig(u) * w;
        }
        y4[v] = make_uint4(pack_bf16(yv[0], yv[1]), pack_bf16(yv[2], yv[3]), pack_bf16(yv[4], yv[5]),
                           pack_bf16(yv[6], yv[7]));
      }
      if (C != nullptr) {
        uint4* u4 = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(C) + row * ldc + col);
        uint4* w4 = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(C) + row * ldc + I + col);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          u4[v] = make_uint4(pack_bf16(__uint_as_float(ru[8 * v]), __uint_as_float(ru[8 * v + 1])),
                             pack_bf16(__uint_as_float(ru[8 * v + 2]), __uint_as_float(ru[8 * v + 3])),
                             pack_bf16(__uint_as_float(ru[8 * v + 4]), __uint_as_float(ru[8 * v + 5])),
                             pack_bf16(__uint_as_float(ru[8 * v + 6]), __uint_as_float(ru[8 * v + 7])));
          w4[v] = make_uint4(pack_bf16(__uint_as_float(rw[8 * v]), __uint_as_float(rw[8 * v + 1])),
                             pack_bf16(__uint_as_float(rw[8 * v + 2]), __uint_as_float(rw[8 * v + 3])),
                             pack_bf16(__uint_as_float(rw[8 * v + 4]), __uint_as_float(rw[8 * v + 5])),
                             pack_bf16(__uint_as_float(rw[8 * v + 6]), __uint_as_float(rw[8 * v + 7])));
        }
      }
    }
  } else if (EPI == EPI_SWIGLU_BWD) {
    // accumulator = dy = dh·Wdown for features nb·BN ..: du = dy·w·σ(u)(1 + u(1−σ(u))), dw = dy·SiLU(u)
    // with u, w read from aux = gu [rows, 2I]; writes C = dgu [rows, 2I]
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(tbase + c, r);
      tmem_wait_ld();
      const int64_t col = static_cast<int64_t>(nb) * BN + c;
      const uint4* gu4 = reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(aux) + row * ldx + col);
      const uint4* gw4 = reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(aux) + row * ldx + I + col);
      uint4* du4 = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(C) + row * ldc + col);
      uint4* dw4 = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(C) + row * ldc + I + col);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint4 ux = gu4[v], wx = gw4[v];
        const bf16* ub = reinterpret_cast<const bf16*>(&ux);
        const bf16* wb = reinterpret_cast<const bf16*>(&wx);
        float du[8], dw[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float u = __bfloat162float(ub[e]), w = __bfloat162float(wb[e]);
          const float dy = __uint_as_float(r[v * 8 + e]);
          const float sg = silu_sig(u);
          du[e] = dy * w * sg * (1.f + u * (1.f - sg));
          dw[e] = dy * u * sg;
        }
        du4[v] = make_uint4(pack_bf16(du[0], du[1]), pack_bf16(du[2], du[3]), pack_bf16(du[4], du[5]),
                            pack_bf16(du[6], du[7]));
        dw4[v] = make_uint4(pack_bf16(dw[0], dw[1]), pack_bf16(dw[2], dw[3]), pack_bf16(dw[4], dw[5]),
                            pack_bf16(dw[6], dw[7]));
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(tbase + c, r);
      tmem_wait_ld();
      const int64_t col = static_cast<int64_t>(nb) * BN + c;
      if (EPI == EPI_BF16) {
        bf16* dst = reinterpret_cast<bf16*>(C) + row * ldc + col;
        float f[32];
  #pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(r[i]);
        if (R != nullptr) {
          const uint4* rs = reinterpret_cast<const uint4*>(R + row * ldc + col);
  #pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 x = rs[v];
            const bf16* xb = reinterpret_cast<const bf16*>(&x);
  #pragma unroll
            for (int i = 0; i < 8; ++i) f[v * 8 + i] += __bfloat162float(xb[i]);
          }
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst);
  #pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 o;
          o.x = pack_bf16(f[v * 8 + 0], f[v * 8 + 1]);
          o.y = pack_bf16(f[v * 8 + 2], f[v * 8 + 3]);
          o.z = pack_bf16(f[v * 8 + 4], f[v * 8 + 5]);
          o.w = pack_bf16(f[v * 8 + 6], f[v * 8 + 7]);
          d4[v] = o;
        }
      } else {
        float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + row * ldc + col);
  #pragma unroll
        for (int v = 0; v < 8; ++v) {
          float4 o = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                 __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
          if (EPI == EPI_F32_ACC) {
            const float4 p = d4[v];
            o.x += p.x;
            o.y += p.y;
            o.z += p.z;
            o.w += p.w;
          }
          d4[v] = o;
        }
      }
    }
  }
}

// Grouped rasterisation of the persistent tile loop (t = linear tile index):
//   raster > 0: bands of `raster` M-tiles sweep over all N-tiles (the A band stays in L2, B streams once per band);
//   raster < 0: bands of −raster N-tiles sweep over all M-tiles (the B band stays in L2, A streams once per band).
// The host picks the orientation and band size that minimise the HBM reads of the operands (choose_raster).
__device__ __forceinline__ void grouped_tile(int t, int num_m, int num_n, int raster, int& mb, int& nb) {
  if (raster > 0) {
    const int group_size = raster * num_n;
    const int first_m = (t / group_size) * raster;
    const int gm = min(raster, num_m - first_m);
    const int r = t % group_size;
    mb = first_m + r % gm;
    nb = r / gm;
  } else {
    const int G = -raster;
    const int group_size = G * num_m;
    const int first_n = (t / group_size) * G;
    const int gn = min(G, num_n - first_n);
    const int r = t % group_size;
    nb = first_n + r % gn;
    mb = r / gn;
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, void* __restrict__ C,
                   int64_t ldc, const bf16* __restrict__ R, int M, int N, int K, void* __restrict__ aux, int64_t ldx,
                   int64_t I, int raster, RopeEpi rope) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + Cfg::STAGES;
  uint64_t* tfull = bars + 2 * Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_m = M / BM, num_n = N / BN, num_k = K / BK;
  const int num_tiles = num_m * num_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int& mb, int& nb) { grouped_tile(t, num_m, num_n, raster, mb, nb); };

  if (warp == 4) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, mb, nb);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          if (!A_MN) {
            tma_load_2d(sa, &tmA, &full[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) tma_load_2d(sa + i * 8192, &tmA, &full[stage], mb * BM + i * 64, kb * BK);
          }
          if (EPI == EPI_SWIGLU_FWD) {  // B tile = 128 gate rows + the matching 128 up rows of [Wgate; Wup]
            tma_load_2d(sb, &tmB, &full[stage], kb * BK, nb * (BN / 2));
            tma_load_2d(sb + (BN / 2) * 128, &tmB, &full[stage], kb * BK, static_cast<int>(I) + nb * (BN / 2));
          } else if (!B_MN) {
            tma_load_2d(sb, &tmB, &full[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(sb + i * 8192, &tmB, &full[stage], nb * BN + i * 64, kb * BK);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(sa + k * 2048, 8192, 1024) : umma_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(sb + k * 2048, 8192, 1024) : umma_desc_sw128(sb + k * 32, 16, 1024);
            umma_f16(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue warps 0..3 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int mb, nb;
      tile_coords(t, mb, nb);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t row = static_cast<int64_t>(mb) * BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      epilogue_tile<BN, EPI>(tbase, row, nb, C, ldc, R, aux, ldx, I, rope);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- CTA-pair variant (cta_group::2)
// A cluster of two CTAs on neighbouring SMs computes one 256×256 output tile with tcgen05.mma.cta_group::2
// (M = 256, N = 256, K = 16), issued by one thread of the even ("leader") CTA.  Each CTA stages only its own 128
// rows of A and its half of the 256 B rows (columns of C), so per SM the smem operand traffic per FLOP and the
// L2 → smem bytes per FLOP both drop by a third against the single-CTA 128×256 tile; each CTA's TMEM holds its
// 128 rows × 256 columns of the accumulator (two accumulators, 512 columns).
//   both CTAs: warp 4 TMA producer into own smem, completion counted on the LEADER's full barrier
//              (the leader's producer posts the expected bytes of both halves);
//              warps 0-3 epilogue on own TMEM, releasing the accumulator on the leader's tempty (8 arrivals)
//   leader:    warp 5 lane 0 issues the pair MMAs; tcgen05.commit multicasts smem-stage release (empty) and
//              accumulator-ready (tfull) to both CTAs
template <int NSTAGE>
struct Gemm2Cfg {
  static constexpr int BN = 256;                      // pair tile N
  static constexpr int STAGES = NSTAGE;
  static constexpr int A_BYTES = BM * BK * 2;         // 16 KB: this CTA's 128 rows of A
  static constexpr int B_BYTES = (BN / 2) * BK * 2;   // 16 KB: this CTA's half of the B tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;
};

template <bool A_MN, bool B_MN, int EPI, int NSTAGE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    void* __restrict__ C, int64_t ldc, const bf16* __restrict__ R, int M, int N, int K,
                    void* __restrict__ aux, int64_t ldx, int64_t I, int raster, int l2hint, RopeEpi rope) {
  using Cfg = Gemm2Cfg<NSTAGE>;
  constexpr int BN = Cfg::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + Cfg::STAGES;
  uint64_t* tfull = bars + 2 * Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int num_m = M / (2 * BM), num_n = N / BN, num_k = K / BK;
  const int num_tiles = num_m * num_n;
  const int cl = blockIdx.x >> 1, n_cl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc_cg2(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();   // barriers of both CTAs initialised before any remote arrival
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int& mb, int& nb) { grouped_tile(t, num_m, num_n, raster, mb, nb); };

  if (warp == 4) {
    if (lane == 0) {
      // l2hint & 3 = 1: the raster keeps an A band resident, 2: a B band -- that operand is loaded evict_last, the
      // streamed one evict_first (l2hint & 4) or evict_normal; 0: evict_normal for both (long-K wgrads)
      const uint64_t last = l2_policy_evict_last(), normal = l2_policy_evict_normal();
      const uint64_t stream = (l2hint & 4) ? l2_policy_evict_first() : normal;
      const uint64_t pol_a = (l2hint & 3) == 1 ? last : (l2hint & 3) ? stream : normal;
      const uint64_t pol_b = (l2hint & 3) == 2 ? last : (l2hint & 3) ? stream : normal;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cl; t < num_tiles; t += n_cl) {
        int mb, nb;
        tile_coords(t, mb, nb);
        const int m0 = mb * 2 * BM + static_cast<int>(rank) * BM;
        const int n0 = EPI == EPI_SWIGLU_FWD ? (rank ? static_cast<int>(I) : 0) + nb * (BN / 2)
                                             : nb * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          const uint32_t bar = mapa_shared(&full[stage], 0);
          if (!A_MN) {
            tma_load_2d_cg2_hint(sa, &tmA, bar, kb * BK, m0, pol_a);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) tma_load_2d_cg2_hint(sa + i * 8192, &tmA, bar, m0 + i * 64, kb * BK, pol_a);
          }
          if (!B_MN) {
            tma_load_2d_cg2_hint(sb, &tmB, bar, kb * BK, n0, pol_b);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 128; ++i)
              tma_load_2d_cg2_hint(sb + i * 8192, &tmB, bar, n0 + i * 64, kb * BK, pol_b);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // drain: every stage's last release (a multicast commit from the leader) has landed before exit
      for (int i = 0; i < Cfg::STAGES; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cl; t < num_tiles; t += n_cl, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(sa + k * 2048, 8192, 1024) : umma_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(sb + k * 2048, 8192, 1024) : umma_desc_sw128(sb + k * 32, 16, 1024);
            umma_f16_cg2(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit_cg2(&empty[stage], 0x3);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_cg2(&tfull[acc], 0x3);
      }
      // drain: both accumulators released by both CTAs' epilogues (remote arrivals landed) before exit
      for (int i = 0; i < 2; ++i, ++it) mbar_wait(&tempty[it & 1], ((it >> 1) & 1) ^ 1);
    }
  } else {
    const int q = warp & 3;
    int it = 0;
    for (int t = cl; t < num_tiles; t += n_cl, ++it) {
      int mb, nb;
      tile_coords(t, mb, nb);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t row = static_cast<int64_t>(mb) * 2 * BM + rank * BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      epilogue_tile<BN, EPI>(tbase, row, nb, C, ldc, R, aux, ldx, I, rope);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    TP_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
    TP_CHECK(q == cudaDriverEntryPointSuccess && p, TAWPIPE_ERUNTIME, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

// 2-D bf16 tensor map: inner dimension `inner` (contiguous), outer dimension `outer` with row pitch `ld`
// elements; box = 64 inner × box_outer, 128-byte swizzle.
CUtensorMap make_tmap_bf16_2d(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TP_CHECK(r == CUDA_SUCCESS, TAWPIPE_ERUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// 2-D fp32 tensor map, box 32 inner (128 B) × box_outer, 128-byte swizzle (used for TMA reduce-add)
CUtensorMap make_tmap_f32_2d(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TP_CHECK(r == CUDA_SUCCESS, TAWPIPE_ERUNTIME, "cuTensorMapEncodeTiled (f32) failed: " + std::to_string((int)r));
  return m;
}

namespace {

int g_num_sms = 0;

// L2-aware raster: keep a band of one operand resident (≤ kL2Band bytes) and stream the other once per band; pick
// the orientation with the fewer estimated HBM operand reads.  Long-K GEMMs (the wgrads, K = tokens) stream K in
// lockstep across the in-flight tiles, so their reuse is per K slice and the default M-band order is kept.
// TAWPIPE_GEMM_RASTER=m|n|default forces an orientation (experiments).
int choose_raster(int64_t num_m, int64_t num_n, int64_t rows_m, int64_t rows_n, int64_t K, int default_group,
                  int* l2hint = nullptr) {
  // l2hint (CTA-pair GEMM): which operand's band the raster keeps resident -- 1 A, 2 B, 0 none (default order),
  // + 4: the streamed operand evict_first.  TAWPIPE_GEMM_L2HINT = 0 (none), 1 (resident evict_last), 2 (+ streamed
  // evict_first) -- experiments
  static const int hints = [] {
    const char* e = std::getenv("TAWPIPE_GEMM_L2HINT");
    return e ? std::atoi(e) : 1;
  }();
  if (l2hint) *l2hint = 0;
  static const int force = [] {
    const char* e = std::getenv("TAWPIPE_GEMM_RASTER");
    if (!e) return 0;
    const std::string v(e);
    return v == "m" ? 1 : v == "n" ? 2 : v == "default" ? 3 : 0;
  }();
  static const int64_t kL2Band = [] {   // resident band budget (TAWPIPE_GEMM_BAND_MB overrides, experiments)
    const char* e = std::getenv("TAWPIPE_GEMM_BAND_MB");
    return (e ? std::atoll(e) : 32ll) << 20;   // measured at the QKV shape: 16 MB 2.76 GB read, 24 1.88, 32 1.72, 48 1.93
  }();
  constexpr int64_t kLongK = 8ll << 20;
  const int64_t bm = rows_m * K * 2, bn = rows_n * K * 2;   // bytes of one M-tile band / one N-tile band
  if (force == 3 || (force == 0 && bm > kLongK && bn > kLongK)) return default_group;
  const int64_t gm = std::max<int64_t>(1, std::min<int64_t>(num_m, kL2Band / bm));
  const int64_t gn = std::max<int64_t>(1, std::min<int64_t>(num_n, kL2Band / bn));
  const int64_t a_bytes = num_m * bm, b_bytes = num_n * bn;
  const int64_t reads_m = a_bytes + b_bytes * ((num_m + gm - 1) / gm);
  const int64_t reads_n = b_bytes + a_bytes * ((num_n + gn - 1) / gn);
  const bool use_n = force == 2 || (force == 0 && reads_n < reads_m);
  if (l2hint && hints) *l2hint = (use_n ? 2 : 1) | (hints >= 2 ? 4 : 0);
  return use_n ? -static_cast<int>(gn) : static_cast<int>(gm);
}

// the dynamic shared-memory limit is a per-device attribute: set it once per (kernel, device)
template <typename K>
void set_smem_attr(K kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert({reinterpret_cast<const void*>(kern), dev}).second)
    TP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

template <int BN, bool A_MN, bool B_MN, int EPI>
void launch(const GemmArgs& g, cudaStream_t s) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, EPI>;
  set_smem_attr(kern, Cfg::SMEM);
  if (g_num_sms == 0) {
    int dev;
    TP_CUDA(cudaGetDevice(&dev));
    TP_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // A: K-major -> rows M, inner K ; MN-major -> inner M, rows K
  CUtensorMap ta = A_MN ? make_tmap_bf16_2d(g.A, g.M, g.K, g.lda, 64) : make_tmap_bf16_2d(g.A, g.K, g.M, g.lda, BM);
  CUtensorMap tb = B_MN ? make_tmap_bf16_2d(g.B, g.N, g.K, g.ldb, 64)
                        : make_tmap_bf16_2d(g.B, g.K, g.N, g.ldb, EPI == EPI_SWIGLU_FWD ? BN / 2 : BN);
  const int tiles = static_cast<int>((g.M / BM) * (g.N / BN));
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  const int raster = choose_raster(g.M / BM, g.N / BN, BM, BN, g.K, 16);
  kern<<<grid, 192, Cfg::SMEM, s>>>(ta, tb, g.C, g.ldc, static_cast<const bf16*>(g.R), static_cast<int>(g.M),
                                     static_cast<int>(g.N), static_cast<int>(g.K), g.aux, g.ldx, g.I, raster, g.rope);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
}

template <int BN, bool A_MN, bool B_MN>
void dispatch_epi(const GemmArgs& g, cudaStream_t s) {
  if (g.epi == 3) {
    if constexpr (!A_MN && !B_MN) launch<BN, A_MN, B_MN, EPI_SWIGLU_FWD>(g, s);
    else throw Error(TAWPIPE_ECONFIG, "SwiGLU forward epilogue needs K-major operands");
  } else if (g.epi == 4) {
    if constexpr (!A_MN && B_MN) launch<BN, A_MN, B_MN, EPI_SWIGLU_BWD>(g, s);
    else throw Error(TAWPIPE_ECONFIG, "SwiGLU backward epilogue is the dgrad form (A K-major, B MN-major)");
  } else if (!g.c_f32)
    launch<BN, A_MN, B_MN, EPI_BF16>(g, s);
  else if (g.accumulate)
    launch<BN, A_MN, B_MN, EPI_F32_ACC>(g, s);
  else
    launch<BN, A_MN, B_MN, EPI_F32_STORE>(g, s);
}

template <int BN>
void dispatch_major(const GemmArgs& g, cudaStream_t s) {
  const bool a_mn = !g.a_kmajor, b_mn = !g.b_kmajor;
  if (!a_mn && !b_mn) dispatch_epi<BN, false, false>(g, s);
  else if (!a_mn && b_mn) dispatch_epi<BN, false, true>(g, s);
  else if (a_mn && b_mn) dispatch_epi<BN, true, true>(g, s);
  else dispatch_epi<BN, true, false>(g, s);
}



template <bool A_MN, bool B_MN, int EPI, int NSTAGE>
void launch2_n(const GemmArgs& g, cudaStream_t s) {
  using Cfg = Gemm2Cfg<NSTAGE>;
  auto kern = gemm_tc2_kernel<A_MN, B_MN, EPI, NSTAGE>;
  static bool attr_set = false;
  static int max_clusters = 0;
  set_smem_attr(kern, Cfg::SMEM);
  if (!attr_set) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 148);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters <= 0) {
      (void)cudaGetLastError();
      max_clusters = 0;
    }
    attr_set = true;
  }
  if (g_num_sms == 0) {
    int dev;
    TP_CUDA(cudaGetDevice(&dev));
    TP_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int clusters_fit = max_clusters > 0 ? max_clusters : g_num_sms / 2;
  CUtensorMap ta = A_MN ? make_tmap_bf16_2d(g.A, g.M, g.K, g.lda, 64) : make_tmap_bf16_2d(g.A, g.K, g.M, g.lda, BM);
  CUtensorMap tb = B_MN ? make_tmap_bf16_2d(g.B, g.N, g.K, g.ldb, 64) : make_tmap_bf16_2d(g.B, g.K, g.N, g.ldb, Cfg::BN / 2);
  const int tiles = static_cast<int>((g.M / (2 * BM)) * (g.N / Cfg::BN));
  const int grid = 2 * (tiles < clusters_fit ? tiles : clusters_fit);
  int l2hint = 0;
  const int raster = choose_raster(g.M / (2 * BM), g.N / Cfg::BN, 2 * BM, Cfg::BN, g.K, 8, &l2hint);
  kern<<<grid, 192, Cfg::SMEM, s>>>(ta, tb, g.C, g.ldc, static_cast<const bf16*>(g.R), static_cast<int>(g.M),
                                     static_cast<int>(g.N), static_cast<int>(g.K), g.aux, g.ldx, g.I, raster, l2hint,
                                     g.rope);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
}

// shared-memory stages of the CTA-pair GEMM: 5 (default; leaves room on the SM for a co-resident NCCL CTA at P > 1)
// or 6 (TAWPIPE_GEMM_STAGES=6).  Same box, C3: 5 stages +0.8 % at N = 1 and +1.1 % at N = 4 in the step, although a
// cold, serialised ncu launch runs ≈10 % slower with 5 (less latency hidden from a cold L2)
template <bool A_MN, bool B_MN, int EPI>
void launch2(const GemmArgs& g, cudaStream_t s) {
  static const int stages = [] {
    const char* e = std::getenv("TAWPIPE_GEMM_STAGES");
    return e ? std::atoi(e) : 5;
  }();
  if (stages == 5)
    launch2_n<A_MN, B_MN, EPI, 5>(g, s);
  else
    launch2_n<A_MN, B_MN, EPI, 6>(g, s);
}

template <bool A_MN, bool B_MN>
void dispatch_epi2(const GemmArgs& g, cudaStream_t s) {
  if (g.epi == 3) {
    if constexpr (!A_MN && !B_MN) launch2<A_MN, B_MN, EPI_SWIGLU_FWD>(g, s);
  } else if (g.epi == 4) {
    if constexpr (!A_MN && B_MN) launch2<A_MN, B_MN, EPI_SWIGLU_BWD>(g, s);
  } else if (!g.c_f32)
    launch2<A_MN, B_MN, EPI_BF16>(g, s);
  else if (g.accumulate)
    launch2<A_MN, B_MN, EPI_F32_ACC>(g, s);
  else
    launch2<A_MN, B_MN, EPI_F32_STORE>(g, s);
}

bool use_pair(const GemmArgs& g) {
  static const int mode = [] {
    const char* e = getenv("TAWPIPE_GEMM_PAIR");
    return e ? atoi(e) : 1;
  }();
  if (mode == 0 || g.M % (2 * BM) != 0 || g.N % 256 != 0) return false;
  if (g.epi == 3 && (g.a_kmajor == false || g.b_kmajor == false)) return false;
  if (g.epi == 4 && !(g.a_kmajor && !g.b_kmajor)) return false;
  return true;
}

void dispatch_pair(const GemmArgs& g, cudaStream_t s) {
  const bool a_mn = !g.a_kmajor, b_mn = !g.b_kmajor;
  if (!a_mn && !b_mn) dispatch_epi2<false, false>(g, s);
  else if (!a_mn && b_mn) dispatch_epi2<false, true>(g, s);
  else if (a_mn && b_mn) dispatch_epi2<true, true>(g, s);
  else dispatch_epi2<true, false>(g, s);
}
}  // namespace

void gemm_tc_bf16(const GemmArgs& g, cudaStream_t s) {
  TP_CHECK(g.M % BM == 0 && g.K % BK == 0 && g.N % 128 == 0, TAWPIPE_ECONFIG,
           "tcgen05 GEMM needs M%128==0, N%128==0, K%64==0 (got " + std::to_string(g.M) + "x" +
               std::to_string(g.N) + "x" + std::to_string(g.K) + ")");
  TP_CHECK(!(g.accumulate && !g.c_f32), TAWPIPE_ECONFIG, "bf16 accumulate-into-C is not supported; use R");
  if (g.epi == 3) {  // the gate/up tile pairs 128 gate rows with 128 up rows: always BN = 256
    TP_CHECK(g.N % 256 == 0 && g.I * 2 == g.N && g.aux, TAWPIPE_ECONFIG, "SwiGLU forward: N = 2I, I % 128 == 0");
    if (use_pair(g)) dispatch_pair(g, s);
    else dispatch_major<256>(g, s);
    return;
  }
  TP_CHECK(!(g.R && g.c_f32), TAWPIPE_ECONFIG, "residual only with bf16 C");
  TP_CHECK(g.rope.cs == nullptr || (g.epi == 0 && !g.c_f32 && !g.R && !g.accumulate && g.rope.dh % 64 == 0 &&
                                    g.rope.cols % 256 == 0 && g.rope.S > 0),
           TAWPIPE_ECONFIG, "RoPE epilogue: bf16 store without residual, d_h % 64 == 0, rotated columns % 256 == 0");
  TP_CHECK((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B) | reinterpret_cast<uintptr_t>(g.C)) %
                   16 == 0 &&
               g.lda % 8 == 0 && g.ldb % 8 == 0 && g.ldc % 8 == 0,
           TAWPIPE_ECONFIG, "tcgen05 GEMM needs 16-byte aligned operands and leading dimensions");
  if (use_pair(g))
    dispatch_pair(g, s);
  else if (g.N % 256 == 0)
    dispatch_major<256>(g, s);
  else
    dispatch_major<128>(g, s);
}

}  // namespace tp
