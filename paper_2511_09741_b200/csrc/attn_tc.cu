// attn_tc.cu -- causal flash attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Computes the causal softmax attention of SURVEY.md §8(c) step 2 (and its backward, §8(c) table) for the
// bf16 path, one (128-row tile, head, sequence) per CTA:
//   forward : S = Q·Kᵀ (TMEM) -> online softmax in registers (exp2, lazily rescaled running max) ->
//             P (bf16, smem) -> O += P·V (TMEM); O / l and LSE written at the end.
//   backward: per 128-row key tile: Sᵀ = K·Qᵀ, dPᵀ = V·dOᵀ (TMEM) -> Pᵀ = exp(Sᵀ − LSE), dSᵀ = Pᵀ⊙(dPᵀ − δ)
//             (bf16, smem) -> dV += Pᵀ·dO, dK += dSᵀ·Q (TMEM, persistent), dQ_i = dS·K (TMEM) reduced into an
//             fp32 accumulator by TMA tensor reduce-add; δ = rowsum(dO⊙O) comes from a pre-pass.
// Causal tiles above the diagonal are skipped (the masked half is work the method avoids, App. B).
// Operand tiles are loaded once by TMA (128 rows × 64 columns, 128-byte swizzle); the same smem tile serves
// as a K-major operand (Q, K for QKᵀ) and as an MN-major operand (V, dO, Q, K in the PV / gradient products).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "ptx.cuh"

namespace tp {

CUtensorMap make_tmap_bf16_2d(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer);
CUtensorMap make_tmap_f32_2d(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer);

namespace {

constexpr int BQ = 128;       // rows per tile (queries or keys)
constexpr int ATOM = 16384;   // one 128-row × 64-col bf16 SW128 tile
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2 / FMUL2: one issue slot for two lanes of work)
__device__ __forceinline__ unsigned long long f2u(float2 a) {
  return (static_cast<unsigned long long>(__float_as_uint(a.y)) << 32) | __float_as_uint(a.x);
}
__device__ __forceinline__ float2 u2f(unsigned long long r) {
  return make_float2(__uint_as_float(static_cast<uint32_t>(r)), __uint_as_float(static_cast<uint32_t>(r >> 32)));
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
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// K-major SW128 descriptor for k-slice ks (16 elements) of a tile made of 64-column atoms
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int ks) {
  return umma_desc_sw128(base + (ks >> 2) * ATOM + (ks & 3) * 32, 16, 1024);
}
// MN-major view of the same storage: K runs over rows (16 rows per slice), MN atoms 16 KB apart
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int ks) {
  return umma_desc_sw128(base + ks * 2048, ATOM, 1024);
}

// =============================================================================================== forward
// ----------------------------------------------------------------------------------------------- forward v3
// One 128-row query tile per CTA; S double-buffered in TMEM, P written back over its S columns (packed bf16)
// and consumed from TMEM as the A operand of O += P·V.  The softmax of tile j therefore never waits for the
// P·V of tile j−1 except when the running max grows by more than 2^8 and O must be rescaled (lazy rescale):
// the exp work overlaps P·V_{j−1} and S_{j+1} on the tensor core.
//   warps 0-3: softmax (thread = row), warp 4: S = Q·Kᵀ issuer, warp 5: P·V issuer, warp 6: TMA producer (Q once;
//   K, V in 3-stage rings).  The MMA issuers run as whole warps (tcgen05.mma from one elected lane, descriptors in
//   uniform registers) and sit on different SMSPs (see the kernel body).
//   TMEM: S0 [0,128) S1 [128,256) O [384,512) (two S/P buffers in flight, see NSB)
template <int DH>
struct Fwd3Smem {
  static constexpr int QB = DH / 64 * ATOM;
  static constexpr int NST = 3;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = QB;
  static constexpr int OFF_V = QB + NST * QB;
  static constexpr int OFF_BAR = QB + 2 * NST * QB;
  static constexpr int BYTES = OFF_BAR + 256;
};

template <int DH>
__global__ void __launch_bounds__(224, 1)
    fa_fwd3_kernel(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, float* __restrict__ lse, int S,
                   int nh, float scale2, unsigned long long* __restrict__ trace) {
  auto TR = [&](int it, int ev) {
    if (trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && it < 32) trace[it * 16 + ev] = clock64();
  };
  using L = Fwd3Smem<DH>;
  constexpr int NST = L::NST;
  // S/P buffers in flight.  Must stay 2: the lazy rescale waits o_done by parity for P·V_{j-1}, which is
  // only unambiguous while S_j being ready implies P·V_{j-2} has completed (S_j is issued after P·V_{j-NSB}).
  // Three buffers measured no faster (r01) and break that invariant.
  constexpr int NSB = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t *q_full = bar, *k_full = bar + 1, *k_empty = bar + 1 + NST, *v_full = bar + 1 + 2 * NST,
           *v_empty = bar + 1 + 3 * NST, *s_full = bar + 1 + 4 * NST, *p_ready = bar + 4 + 4 * NST,
           *o_done = bar + 7 + 4 * NST, *pv_done = bar + 8 + 4 * NST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10 + 4 * NST);

  const int n_q = S / BQ;
  // head-major order (the K/V of one head stay in L2 across its query tiles), heaviest tiles first in a head
  const int qt = n_q - 1 - static_cast<int>(blockIdx.x % n_q);
  const int h = static_cast<int>(blockIdx.x / n_q);
  const int b = blockIdx.y;
  const int H = nh * DH;
  const int row0 = b * S;
  const int n_kv = qt + 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    if (smem_u32(sm) & 1023) __trap();
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < NSB; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_ready[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 384;   // S/P buffers at 0 and 128

  // The two MMA chains are issued from different SMSPs: an SMSP that issues tcgen05.mma loses roughly the MMAs'
  // execution time of issue slots (measured: the softmax warp sharing the issuer's SMSP finished each tile ~1000
  // cycles late with both chains on one warp), so the S chain (warp 4, SMSP 0) and the P·V chain (warp 5,
  // SMSP 1) each cost their neighbour half of that; the TMA producer is warp 6 (SMSP 2).
  if (warp == 6) {
    if (lane == 0) {
      mbar_expect_tx(q_full, L::QB);
      for (int a = 0; a < DH / 64; ++a)
        tma_load_2d(sm + L::OFF_Q + a * ATOM, &tm, q_full, h * DH + a * 64, row0 + qt * BQ);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % NST;
        const uint32_t ph = (j / NST) & 1;
        mbar_wait_sleep(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], L::QB);
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sm + L::OFF_K + st * L::QB + a * ATOM, &tm, &k_full[st], H + h * DH + a * 64, row0 + j * BQ);
        mbar_wait_sleep(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], L::QB);
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sm + L::OFF_V + st * L::QB + a * ATOM, &tm, &v_full[st], 2 * H + h * DH + a * 64,
                      row0 + j * BQ);
      }
    }
  } else if (warp == 4) {
    // S chain: S_j = Q·K_jᵀ into buffer j % 2 once P·V_{j−2} (the previous reader of that buffer) completed
    constexpr uint32_t id_qk = umma_idesc_bf16(128, 128, false, false);
    const uint32_t sQ = smem_u32(sm + L::OFF_Q);
    mbar_wait_sleep(q_full, 0);
    for (int j = 0; j < n_kv; ++j) {
      const int st = j % NST;
      if (j >= NSB) mbar_wait_sleep(&pv_done[j % NSB], ((j - NSB) / NSB) & 1);
      mbar_wait_sleep(&k_full[st], (j / NST) & 1);
      tc_fence_after();
      const uint32_t sK = smem_u32(sm + L::OFF_K + st * L::QB);
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks)
        umma_f16_w(tmem + (j % NSB) * 128, desc_k(sQ, ks), desc_k(sK, ks), id_qk, ks > 0);
      umma_commit_w(&k_empty[st]);
      umma_commit_w(&s_full[j % NSB]);
    }
  } else if (warp == 5) {
    // P·V chain: O += P_j·V_j with P_j (bf16) read from TMEM as the A operand
    constexpr uint32_t id_pv = umma_idesc_bf16(128, DH, false, true);
    for (int j = 0; j < n_kv; ++j) {
      const int st = j % NST;
      mbar_wait_sleep(&p_ready[j % NSB], (j / NSB) & 1);
      TR(j, 0);
      mbar_wait_sleep(&v_full[st], (j / NST) & 1);
      TR(j, 1);
      tc_fence_after();
      const uint32_t sV = smem_u32(sm + L::OFF_V + st * L::QB);
#pragma unroll
      for (int ks = 0; ks < BQ / 16; ++ks)
        umma_f16_tmemA_w(tO, tmem + (j % NSB) * 128 + ks * 8, desc_mn(sV, ks), id_pv, (j | ks) > 0);
      umma_commit_w(&v_empty[st]);
      umma_commit_w(&pv_done[j % NSB]);
      umma_commit_w(o_done);
      TR(j, 2);
    }
  } else {
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    float m2 = -INFINITY, l = 0.f;
    float s[128];
    for (int j = 0; j < n_kv; ++j) {
      const uint32_t tS = tmem + (j % NSB) * 128 + lane_off;
      mbar_wait(&s_full[j % NSB], (j / NSB) & 1);
      if (r == 0) TR(j, 3);
      tc_fence_after();
      {  // all four loads in flight before one wait (one TMEM round trip per row)
        uint32_t u0[32], u1[32], u2[32], u3[32];
        tmem_ld32(tS, u0);
        tmem_ld32(tS + 32, u1);
        tmem_ld32(tS + 64, u2);
        tmem_ld32(tS + 96, u3);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = __uint_as_float(u0[i]);
          s[32 + i] = __uint_as_float(u1[i]);
          s[64 + i] = __uint_as_float(u2[i]);
          s[96 + i] = __uint_as_float(u3[i]);
        }
      }
      if (j == qt) {  // diagonal tile only
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i > r) s[i] = -INFINITY;
      }
      // row max with 8 independent chains (one softmax warp per SMSP: latency is not hidden)
      float mxa[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mxa[k] = s[k];
#pragma unroll
      for (int i = 8; i < 128; ++i) mxa[i & 7] = fmaxf(mxa[i & 7], s[i]);
      float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                       fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
      mx *= scale2;
      if (j == 0) {
        m2 = mx;
      } else if (__any_sync(0xffffffffu, mx > m2 + 8.0f)) {
        // rescale O: needs P·V_{j-1} complete (the only place the softmax waits for the tensor core)
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
        const float mnew = fmaxf(m2, mx);
        const float alpha = ex2(m2 - mnew);
        l *= alpha;
#pragma unroll 1
        for (int c = 0; c < DH / 32; ++c) {
          uint32_t u[32];
          tmem_ld32(tO + lane_off + c * 32, u);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
          tmem_st32(tO + lane_off + c * 32, u);
        }
        m2 = mnew;
      }
      float2 sa2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 sc2 = make_float2(scale2, scale2), nm2 = make_float2(-m2, -m2);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pw[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 a2 = ffma2(make_float2(s[c * 32 + i], s[c * 32 + i + 1]), sc2, nm2);
          const float p0 = ex2(a2.x);
          const float p1 = ex2(a2.y);
          sa2[(i >> 1) & 3] = fadd2(sa2[(i >> 1) & 3], make_float2(p0, p1));
          pw[i / 2] = pack_bf16(p0, p1);
        }
        tmem_st16(tS + c * 16, pw);
      }
      const float2 t2 = fadd2(fadd2(sa2[0], sa2[1]), fadd2(sa2[2], sa2[3]));
      l += t2.x + t2.y;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_ready[j % NSB]);
      if (lane == 0) TR(j, 4 + q);   // per-warp p_done (slots 4..7)
    }
    mbar_wait(o_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    bf16* orow = out + static_cast<int64_t>(row0 + qt * BQ + r) * H + h * DH;
#pragma unroll 1
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t u[32];
      tmem_ld32(tO + lane_off + c * 32, u);
      tmem_wait_ld();
      uint4* d4 = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 o;
        o.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * inv, __uint_as_float(u[8 * v + 1]) * inv);
        o.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv);
        o.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv);
        o.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv);
        d4[v] = o;
      }
    }
    lse[(static_cast<int64_t>(b) * nh + h) * S + qt * BQ + r] = (m2 + __log2f(l)) * (1.0f / LOG2E);
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int DH>
struct Fwd5Smem {
  static constexpr int QB = DH / 64 * ATOM;
  static constexpr int NST = 2;
  static constexpr int OFF_Q = 0;   // Q_A, Q_B
  static constexpr int OFF_K = 2 * QB;
  static constexpr int OFF_V = 2 * QB + NST * QB;
  static constexpr int OFF_BAR = 2 * QB + 2 * NST * QB;
  static constexpr int BYTES = OFF_BAR + 256;
};
// ----------------------------------------------------------------------------------------------- forward v7
// Two query tiles per CTA (A = 2p+1, B = 2p: one K/V stream, A one key tile longer), one softmax warpgroup each
// (thread = row), so one tile's exponentials run on the MUFU while the other tile's scores are loaded, reduced and
// written back (the r01 "v5" design, superseded by this kernel and removed).  Every 128-key step is
// processed as two 64-key halves with their own online-softmax update: S_t(j, half) is an N = 64 MMA, P_t(j, half)
// goes back over the first 32 columns of its half, P·V_t(j, half) is a K = 64 MMA, and S_t(j+1, half) is issued
// right behind it.  A tile's softmax therefore works on one half while the tensor core runs the other half's P·V
// and next S, instead of waiting for a whole P·V + S after each 128-key step (measured ≈2,050 cycles per step in
// v5).  One issuer warp per tile keeps the two tiles' MMA streams independent.  Sustained at S = 32K, 32 heads:
// 7.35 ms against v5's 8.4 ms (7.9 ms with a single in-order issuer for both tiles).
//   TMEM per tile t: S/P [128t, 128t+128) as halves of 64 columns, O_t [256+128t, 384+128t)
template <int DH>
__global__ void __launch_bounds__(384, 1)
    fa_fwd7_kernel(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, float* __restrict__ lse, int S,
                   int nh, float scale2) {
  using L = Fwd5Smem<DH>;
  constexpr int NST = L::NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t *q_full = bar, *k_full = bar + 1, *k_empty = bar + 1 + NST, *v_full = bar + 1 + 2 * NST,
           *v_empty = bar + 1 + 3 * NST;
  uint64_t* s_full = bar + 1 + 4 * NST;    // [tile][half]
  uint64_t* p_ready = bar + 5 + 4 * NST;   // [tile][half]
  uint64_t* o_done = bar + 9 + 4 * NST;    // [tile]: one phase per P·V half
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 11 + 4 * NST);

  const int n_pairs = S / BQ / 2;
  const int pr = n_pairs - 1 - static_cast<int>(blockIdx.x % n_pairs);
  const int h = static_cast<int>(blockIdx.x / n_pairs);
  const int b = blockIdx.y;
  const int H = nh * DH;
  const int row0 = b * S;
  const int n_kv_A = 2 * pr + 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    if (smem_u32(sm) & 1023) __trap();
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 2);   // released by both tiles' issuers (the last K / V only by tile A's: not reused)
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 2);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_ready[i], 128);
    }
    mbar_init(&o_done[0], 1);
    mbar_init(&o_done[1], 1);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc(tmem_slot, 512);   // warps 0-7 softmax, 8 / 10 issuers, 9 producer
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 9) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * L::QB);
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sm + L::OFF_Q + t * L::QB + a * ATOM, &tm, q_full, h * DH + a * 64,
                      row0 + (2 * pr + 1 - t) * BQ);
      for (int j = 0; j < n_kv_A; ++j) {
        const int st = j % NST;
        const uint32_t ph = (j / NST) & 1;
        mbar_wait_sleep(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], L::QB);
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sm + L::OFF_K + st * L::QB + a * ATOM, &tm, &k_full[st], H + h * DH + a * 64, row0 + j * BQ);
        mbar_wait_sleep(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], L::QB);
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sm + L::OFF_V + st * L::QB + a * ATOM, &tm, &v_full[st], 2 * H + h * DH + a * 64,
                      row0 + j * BQ);
      }
    }
  } else if (warp == 8 || warp == 10) {
    // one in-order issuer per tile (warp 8: A on SMSP 0, warp 10: B on SMSP 2): P·V_t(j, half) then S_t(j+1, half),
    // so that a tile's MMAs never queue behind the other tile's softmax
    const int t = warp == 8 ? 0 : 1;
    const int n_kv_t = n_kv_A - t;
    constexpr uint32_t id_qk = umma_idesc_bf16(128, 64, false, false);
    constexpr uint32_t id_pv = umma_idesc_bf16(128, DH, false, true);
    const uint32_t sQ = smem_u32(sm + L::OFF_Q + t * L::QB);
    auto issue_s = [&](int jj, int hf) {   // S_t(jj, hf) = Q_t · K_jj[64·hf .. 64·hf+63]ᵀ (N = 64)
      const uint32_t sK = smem_u32(sm + L::OFF_K + (jj % NST) * L::QB) + hf * 8192;
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks)
        umma_f16_w(tmem + t * 128 + hf * 64, desc_k(sQ, ks), desc_k(sK, ks), id_qk, ks > 0);
      umma_commit_w(&s_full[t * 2 + hf]);
    };
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(0, 1);
    umma_commit_w(&k_empty[0]);
    for (int j = 0; j < n_kv_t; ++j) {
      const int st = j % NST;
      mbar_wait(&v_full[st], (j / NST) & 1);
      const uint32_t sV = smem_u32(sm + L::OFF_V + st * L::QB);
      const bool next = j + 1 < n_kv_t;
      if (next) mbar_wait(&k_full[(j + 1) % NST], ((j + 1) / NST) & 1);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        mbar_wait(&p_ready[t * 2 + hf], j & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)   // keys 64·hf + 16·ks: P packed over the half's first 32 columns
          umma_f16_tmemA_w(tmem + 256 + t * 128, tmem + t * 128 + hf * 64 + ks * 8, desc_mn(sV, hf * 4 + ks), id_pv,
                           (j | hf | ks) > 0);
        umma_commit_w(&o_done[t]);
        if (next) issue_s(j + 1, hf);
      }
      umma_commit_w(&v_empty[st]);
      if (next) umma_commit_w(&k_empty[(j + 1) % NST]);
    }
  } else {
    const int t = warp >> 2;          // 0: tile A, 1: tile B
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int qt = 2 * pr + 1 - t;
    const int n_kv = qt + 1;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tO = tmem + 256 + t * 128 + lane_off;
    float m2 = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        const uint32_t tS = tmem + t * 128 + hf * 64 + lane_off;
        mbar_wait(&s_full[t * 2 + hf], j & 1);
        tc_fence_after();
        float s[64];
        {
          uint32_t u0[32], u1[32];
          tmem_ld32(tS, u0);
          tmem_ld32(tS + 32, u1);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            s[i] = __uint_as_float(u0[i]);
            s[32 + i] = __uint_as_float(u1[i]);
          }
        }
        if (j == qt) {  // diagonal tile only: key 64·hf + i > row r is masked
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (hf * 64 + i > r) s[i] = -INFINITY;
        }
        float mxa[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mxa[k] = s[k];
#pragma unroll
        for (int i = 8; i < 64; ++i) mxa[i & 7] = fmaxf(mxa[i & 7], s[i]);
        float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                         fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        mx *= scale2;
        if (j == 0 && hf == 0) {
          m2 = mx;
        } else if (__any_sync(0xffffffffu, mx > m2 + 8.0f)) {
          // lazy rescale: O_t must hold exactly the P·V halves issued so far (phase 2j + hf − 1 of o_done[t];
          // the one before it completed with S_t(j, hf), so the parity wait is unambiguous)
          mbar_wait(&o_done[t], (2 * j + hf - 1) & 1);
          tc_fence_after();
          const float mnew = fmaxf(m2, mx);
          const float alpha = ex2(m2 - mnew);
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t u[32];
            tmem_ld32(tO + c * 32, u);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
            tmem_st32(tO + c * 32, u);
          }
          m2 = mnew;
        }
        float2 sa2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sc2 = make_float2(scale2, scale2), nm2 = make_float2(-m2, -m2);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pw[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 a2 = ffma2(make_float2(s[c * 32 + i], s[c * 32 + i + 1]), sc2, nm2);
            const float p0 = ex2(a2.x), p1 = ex2(a2.y);
            sa2[(i >> 1) & 3] = fadd2(sa2[(i >> 1) & 3], make_float2(p0, p1));
            pw[i / 2] = pack_bf16(p0, p1);
          }
          tmem_st16(tS + c * 16, pw);
        }
        const float2 t2 = fadd2(fadd2(sa2[0], sa2[1]), fadd2(sa2[2], sa2[3]));
        l += t2.x + t2.y;
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_ready[t * 2 + hf]);
      }
    }
    // the last two P·V halves (phases 2·n_kv − 2 and 2·n_kv − 1), waited in order so that each parity is unambiguous
    mbar_wait(&o_done[t], 0);
    mbar_wait(&o_done[t], 1);
    tc_fence_after();
    const float inv = 1.f / l;
    bf16* orow = out + static_cast<int64_t>(row0 + qt * BQ + r) * H + h * DH;
#pragma unroll 1
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t u[32];
      tmem_ld32(tO + c * 32, u);
      tmem_wait_ld();
      uint4* d4 = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 o;
        o.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * inv, __uint_as_float(u[8 * v + 1]) * inv);
        o.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv);
        o.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv);
        o.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv);
        d4[v] = o;
      }
    }
    lse[(static_cast<int64_t>(b) * nh + h) * S + qt * BQ + r] = (m2 + __log2f(l)) * (1.0f / LOG2E);
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// =============================================================================================== backward
// Warp roles (320 threads, one CTA per SM):
//   warps 0-3  softmax-gradient warps, thread t <-> key row t of the tile (TMEM lane t):
//              Pᵀ = exp2(Sᵀ·c·log2e − LSE·log2e) is written back into TMEM as packed bf16 over Sᵀ's columns
//              (the A operand of dV += Pᵀ·dO), dSᵀ = Pᵀ⊙(dPᵀ − δ) goes to smem (A of dK, MN-major A of dQ)
//   warps 4-7  dQ warps: read dQ_i (TMEM lanes = query rows) into registers, stage it (fp32, 128-byte
//              swizzle) in a dedicated smem buffer and add it into the fp32 accumulator with TMA tensor
//              reduce-add (cp.reduce.async.bulk.tensor) -- the L2 reduction runs off the critical path
//   warp 8     TMA producer: K, V once; Q_i (+ LSE_i, δ_i by bulk copy) double-buffered; dO_i single-buffered
//              (released as soon as dV += Pᵀ·dO has consumed it)
//   warp 9     MMA issuer: Sᵀ, dPᵀ, dV, dK, dQ_i (into dPᵀ's TMEM columns)
//   TMEM: Sᵀ/Pᵀ [0,128) dPᵀ/dQ [128,256) dV [256,256+d) dK [256+d,256+2d)
template <int DH>
struct BwdSmem {
  static constexpr int QB = DH / 64 * ATOM;
  static constexpr int OFF_K = 0, OFF_V = QB, OFF_Q = 2 * QB, OFF_DO = 4 * QB;  // Q: 2 stages, dO: 1
  static constexpr int OFF_DS = 5 * QB;              // dSᵀ [kv][q], 2 atoms
  static constexpr int OFF_STG = OFF_DS + 2 * ATOM;  // dQ staging: 2 × (128 rows × 32 fp32) per round
  static constexpr int OFF_LSE = OFF_STG + 2 * ATOM; // 2 stages × 128 floats
  static constexpr int OFF_DEL = OFF_LSE + 1024;     // 2 stages × 128 floats
  static constexpr int OFF_BAR = OFF_DEL + 1024;
  static constexpr int BYTES = OFF_BAR + 256;
};

__device__ __forceinline__ float bf_lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf_hi(uint32_t x) { return __uint_as_float(x & 0xFFFF0000u); }

template <int DH>
__global__ void __launch_bounds__(384, 1)   // 352 threads; 168 registers (three warps share SMSPs 0-2)
    fa_bwd_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmdo,
                  const __grid_constant__ CUtensorMap tmdq, const float* __restrict__ lse,
                  const float* __restrict__ delta, float* __restrict__ dq_acc, bf16* __restrict__ dqkv, int S, int nh,
                  float scale, float scale2, unsigned long long* __restrict__ trace, const float* __restrict__ rcos,
                  const float* __restrict__ rsin) {
  using L = BwdSmem<DH>;
  // debug timeline (CTA 0 only, first 32 iterations): trace[it * 16 + event] = clock64()
  auto TR = [&](int it, int ev) {
    if (trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && it < 32) trace[it * 16 + ev] = clock64();
  };
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t *kv_full = bar, *q_full = bar + 1, *q_empty = bar + 3, *do_full = bar + 5, *do_empty = bar + 6,
           *s_full = bar + 7, *dp_full = bar + 8, *tdp_free = bar + 9, *p_ready = bar + 10, *ds_ready = bar + 11,
           *mm2_done = bar + 12, *dq_done = bar + 13, *dv_done = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);
  float* lse_s = reinterpret_cast<float*>(sm + L::OFF_LSE);
  float* del_s = reinterpret_cast<float*>(sm + L::OFF_DEL);

  const int n_q = S / BQ;
  // head-major order (Q, dO of one head stay in L2), heaviest key tiles (most query tiles) first in a head
  const int jt = static_cast<int>(blockIdx.x % n_q);
  const int h = static_cast<int>(blockIdx.x / n_q);
  const int b = blockIdx.y;
  const int H = nh * DH;
  const int row0 = b * S;
  const int n_it = n_q - jt;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    if (smem_u32(sm) & 1023) __trap();  // SW128 tiles need a 1024-byte aligned base
    tma_prefetch(&tm);
    tma_prefetch(&tmdo);
    tma_prefetch(&tmdq);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(tdp_free, 128);
    mbar_init(p_ready, 128);
    mbar_init(ds_ready, 128);
    mbar_init(mm2_done, 1);
    mbar_init(dq_done, 1);
    mbar_init(dv_done, 1);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + DH;

  if (warp == 8) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * L::QB);
      for (int a = 0; a < DH / 64; ++a) {
        tma_load_2d(sm + L::OFF_K + a * ATOM, &tm, kv_full, H + h * DH + a * 64, row0 + jt * BQ);
        tma_load_2d(sm + L::OFF_V + a * ATOM, &tm, kv_full, 2 * H + h * DH + a * 64, row0 + jt * BQ);
      }
      for (int it = 0; it < n_it; ++it) {
        const int i = jt + it, st = it & 1;
        mbar_wait(&q_empty[st], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[st], L::QB + 1024);
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sm + L::OFF_Q + st * L::QB + a * ATOM, &tm, &q_full[st], h * DH + a * 64, row0 + i * BQ);
        const int64_t li = (static_cast<int64_t>(b) * nh + h) * S + i * BQ;
        bulk_load(lse_s + st * 128, lse + li, 512, &q_full[st]);
        bulk_load(del_s + st * 128, delta + li, 512, &q_full[st]);
        mbar_wait(do_empty, (it & 1) ^ 1);
        mbar_expect_tx(do_full, L::QB);
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sm + L::OFF_DO + a * ATOM, &tmdo, do_full, h * DH + a * 64, row0 + i * BQ);
      }
    }
  } else if (warp == 9 || warp == 10) {
    // two MMA issuers on SMSPs 1 and 2, each a whole warp with one elected lane issuing:
    //   warp 9  (X): dPᵀ_i (after dQ_{i−1} was drained), then Sᵀ_{i+1} (after dV_i has read Pᵀ_i)
    //   warp 10 (Y): dV_i (after Pᵀ_i is written), then dQ_i, dK_i (after dSᵀ_i is in smem)
    // an SMSP that issues MMAs loses issue slots to its other warps roughly while they execute: splitting the five
    // products over two SMSPs halves what the compute warp sharing each one loses
    constexpr uint32_t id_s = umma_idesc_bf16(128, 128, false, false);  // Sᵀ, dPᵀ: K = d
    constexpr uint32_t id_kv = umma_idesc_bf16(128, DH, false, true);   // dV, dK: A K-major (K = q), B MN-major
    constexpr uint32_t id_q = umma_idesc_bf16(128, DH, true, true);     // dQ: A = dSᵀ viewed MN-major
    const uint32_t sK = smem_u32(sm + L::OFF_K), sV = smem_u32(sm + L::OFF_V), sDS = smem_u32(sm + L::OFF_DS),
                   sDO = smem_u32(sm + L::OFF_DO);
    if (warp == 9) {
      auto issue_s = [&](int it) {  // Sᵀ_it = K·Q_itᵀ into tS
        const int st = it & 1;
        mbar_wait(&q_full[st], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(sm + L::OFF_Q + st * L::QB);
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) umma_f16_w(tS, desc_k(sK, ks), desc_k(sQ, ks), id_s, ks > 0);
        umma_commit_w(s_full);
        TR(it, 0);
      };
      mbar_wait(kv_full, 0);
      issue_s(0);
      for (int it = 0; it < n_it; ++it) {
        mbar_wait(do_full, it & 1);
        if (it > 0) mbar_wait(tdp_free, (it - 1) & 1);
        TR(it, 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) umma_f16_w(tdP, desc_k(sV, ks), desc_k(sDO, ks), id_s, ks > 0);
        umma_commit_w(dp_full);
        if (it + 1 < n_it) {
          mbar_wait(dv_done, it & 1);   // Sᵀ_{it+1} overwrites Pᵀ_it: only after dV_it has read it
          issue_s(it + 1);
        }
      }
    } else {
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1;
        const uint32_t sQ = smem_u32(sm + L::OFF_Q + st * L::QB);
        mbar_wait(p_ready, it & 1);
        mbar_wait(dp_full, it & 1);    // dPᵀ_it (issuer X) has read dO_i before dO is released below
        TR(it, 2);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks) umma_f16_tmemA_w(tdV, tS + ks * 8, desc_mn(sDO, ks), id_kv, (it | ks) > 0);
        umma_commit_w(do_empty);
        umma_commit_w(dv_done);
        mbar_wait(ds_ready, it & 1);
        TR(it, 3);
        // dQ_it precedes dK_it: its drain (which frees the TMEM columns dPᵀ_{it+1} needs) overlaps dK_it
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks) umma_f16_w(tdP, desc_mn(sDS, ks), desc_mn(sK, ks), id_q, ks > 0);
        umma_commit_w(dq_done);
#pragma unroll
        for (int ks = 0; ks < BQ / 16; ++ks) umma_f16_w(tdK, desc_k(sDS, ks), desc_mn(sQ, ks), id_kv, (it | ks) > 0);
        umma_commit_w(&q_empty[st]);
        umma_commit_w(mm2_done);
      }
    }
  } else if (warp < 4) {
    const int t = warp * 32 + lane;  // key row of the tile (TMEM lane)
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    uint8_t* sDS = sm + L::OFF_DS;
    for (int it = 0; it < n_it; ++it) {
      const int st = it & 1;
      const float* ls = lse_s + st * 128;
      const float* dl = del_s + st * 128;
      mbar_wait(&q_full[st], (it >> 1) & 1);   // LSE_i, δ_i landed (bulk copies on the same barrier as Q_i)
      mbar_wait(s_full, it & 1);
      if (t == 0) TR(it, 4);
      tc_fence_after();
      // ls holds LSE·log2(e) (pre-scaled by the δ kernel); the diagonal tile (it == 0) takes the masked path
      uint32_t pk[4][16];   // Pᵀ_it, packed bf16, kept for the dS pass (Sᵀ_{it+1} overwrites its TMEM copy)
      auto p_pass = [&](auto diag) {
#pragma unroll
        for (int cp = 0; cp < 4; cp += 2) {  // two chunks per TMEM round trip
          uint32_t uu[2][32];
          tmem_ld32(tS + lane_off + cp * 32, uu[0]);
          tmem_ld32(tS + lane_off + cp * 32 + 32, uu[1]);
          tmem_wait_ld();
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int c = cp + h2;
            uint32_t (&pw)[16] = pk[c];
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              const float2 l2 = *reinterpret_cast<const float2*>(ls + c * 32 + k);
              const float2 a2 = ffma2(make_float2(__uint_as_float(uu[h2][k]), __uint_as_float(uu[h2][k + 1])),
                                      make_float2(scale2, scale2), make_float2(-l2.x, -l2.y));
              float p0 = ex2(a2.x);
              float p1 = ex2(a2.y);
              if (decltype(diag)::value) {  // query index < key index is masked
                if (c * 32 + k < t) p0 = 0.f;
                if (c * 32 + k + 1 < t) p1 = 0.f;
              }
              pw[k / 2] = pack_bf16(p0, p1);
            }
            tmem_st16(tS + lane_off + c * 16, pw);  // overwrites Sᵀ columns already read (c*16 < cp*32+64)
          }
        }
      };
      if (it == 0)
        p_pass(std::true_type{});
      else
        p_pass(std::false_type{});
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_ready);
      if (t == 0) TR(it, 5);
      mbar_wait(dp_full, it & 1);
      if (t == 0) TR(it, 6);
      if (it > 0) mbar_wait(mm2_done, (it - 1) & 1);  // dSᵀ of the previous tile consumed by dK / dQ
      if (t == 0) TR(it, 7);
      tc_fence_after();
#pragma unroll
      for (int cp = 0; cp < 4; cp += 2) {  // two chunks per TMEM round trip
        uint32_t uu[2][32];
        tmem_ld32(tdP + lane_off + cp * 32, uu[0]);
        tmem_ld32(tdP + lane_off + cp * 32 + 32, uu[1]);
        tmem_wait_ld();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c = cp + h2;
          const uint32_t (&pp)[16] = pk[c];
          uint32_t d[16];
#pragma unroll
          for (int k = 0; k < 32; k += 2) {
            const float2 dl2 = *reinterpret_cast<const float2*>(dl + c * 32 + k);
            const float2 ds2 = fmul2(make_float2(bf_lo(pp[k / 2]), bf_hi(pp[k / 2])),
                                     fadd2(make_float2(__uint_as_float(uu[h2][k]), __uint_as_float(uu[h2][k + 1])),
                                           make_float2(-dl2.x, -dl2.y)));
            d[k / 2] = pack_bf16(ds2.x, ds2.y);
          }
          // 32 columns = 4 × 16-byte chunks of atom c/2, chunk index (c%2)*4 + v
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int chunk = (c & 1) * 4 + v;
            *reinterpret_cast<uint4*>(sDS + (c >> 1) * ATOM + t * 128 + ((chunk ^ (t & 7)) << 4)) =
                make_uint4(d[4 * v], d[4 * v + 1], d[4 * v + 2], d[4 * v + 3]);
          }
        }
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(ds_ready);
      if (t == 0) TR(it, 8);
      if (lane == 0) TR(it, 12 + warp);   // per-warp dS done
    }
    // dK (× softmax scale) and dV rows of this key tile.  With RoPE tables (rcos != nullptr) dK is also rotated back
    // by −p·θ_i (the inverse RoPE of the step: dk_i = dy_i cos + dy_{i+d/2} sin, dk_{i+d/2} =
    // dy_{i+d/2} cos − dy_i sin), so no separate pass re-reads dqkv: columns c and c + d/2 are loaded together.
    mbar_wait(mm2_done, (n_it - 1) & 1);
    tc_fence_after();
    bf16* dkp = dqkv + static_cast<int64_t>(row0 + jt * BQ + t) * 3 * H + H + h * DH;
    bf16* dvp = dkp + H;
    auto st32 = [&](bf16* dst, const float* f) {   // 32 fp32 -> 32 bf16, four 16-byte stores
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        d4[v] = make_uint4(pack_bf16(f[8 * v + 0], f[8 * v + 1]), pack_bf16(f[8 * v + 2], f[8 * v + 3]),
                           pack_bf16(f[8 * v + 4], f[8 * v + 5]), pack_bf16(f[8 * v + 6], f[8 * v + 7]));
    };
#pragma unroll 1
    for (int c = 0; c < DH / 32; ++c) {   // dV
      uint32_t w[32];
      tmem_ld32(tdV + lane_off + c * 32, w);
      tmem_wait_ld();
      float f[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(w[e]);
      st32(dvp + c * 32, f);
    }
    constexpr int HALF = DH / 2;
    const float* cpos = rcos ? rcos + static_cast<int64_t>(jt * BQ + t) * HALF : nullptr;
    const float* spos = rsin ? rsin + static_cast<int64_t>(jt * BQ + t) * HALF : nullptr;
#pragma unroll 1
    for (int c = 0; c < HALF / 32; ++c) {   // dK: chunk c of the first half with chunk c of the second half
      uint32_t u1[32], u2[32];
      tmem_ld32(tdK + lane_off + c * 32, u1);
      tmem_ld32(tdK + lane_off + HALF + c * 32, u2);
      tmem_wait_ld();
      float a[32], b2[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        a[e] = __uint_as_float(u1[e]) * scale;
        b2[e] = __uint_as_float(u2[e]) * scale;
      }
      if (cpos) {
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 cc = reinterpret_cast<const float4*>(cpos + c * 32)[q4];
          const float4 ss = reinterpret_cast<const float4*>(spos + c * 32)[q4];
          const float cv[4] = {cc.x, cc.y, cc.z, cc.w}, sv[4] = {ss.x, ss.y, ss.z, ss.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x1 = a[4 * q4 + e], x2 = b2[4 * q4 + e];
            a[4 * q4 + e] = x1 * cv[e] + x2 * sv[e];
            b2[4 * q4 + e] = x2 * cv[e] - x1 * sv[e];
          }
        }
      }
      st32(dkp + c * 32, a);
      st32(dkp + HALF + c * 32, b2);
    }
    tc_fence_before();
  } else if (warp < 8) {
    // dQ warps 4-7: TMEM lane quarter (warp % 4) holds query rows of dQ_i
    const int q = warp & 3;
    const int t = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    uint8_t* stg = sm + L::OFF_STG;
    int rnd = 0;   // staging rounds issued so far (buffer half = rnd & 1)
    for (int it = 0; it < n_it; ++it) {
      const int i = jt + it;
      mbar_wait(dq_done, it & 1);    // dQ_i complete
      if (t == 0) TR(it, 9);
      tc_fence_after();
      uint32_t u[DH / 32][32];
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) tmem_ld32(tdP + lane_off + c * 32, u[c]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(tdp_free);                   // TMEM columns free for the next dPᵀ
      if (t == 0) TR(it, 10);
      // 32-column rounds through the two 16 KB halves of the staging buffer: a round waits only for the reduce
      // issued two rounds earlier (wait_group.read 1), so writing one half overlaps the TMA read of the other
#pragma unroll
      for (int c = 0; c < DH / 32; ++c, ++rnd) {
        uint8_t* buf = stg + (rnd & 1) * ATOM;
        if (t == 0) bulk_wait_read1();
        named_bar(2, 128);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(buf + t * 128 + ((j ^ (t & 7)) << 4)) =
              make_uint4(u[c][4 * j], u[c][4 * j + 1], u[c][4 * j + 2], u[c][4 * j + 3]);
        fence_async_smem();
        named_bar(2, 128);
        if (t == 0) {
          tma_reduce_add_2d(&tmdq, buf, h * DH + c * 32, row0 + i * BQ);
          bulk_commit();
        }
      }
      if (t == 0) TR(it, 11);
    }
    if (t == 0) bulk_wait_all0();
  }
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


// δ_i = Σ_d dO_id·O_id ; one warp per (row, head)
__global__ void fa_delta_kernel(int64_t rows, int S, int nh, int dh, const bf16* __restrict__ o,
                                const bf16* __restrict__ dout, float* __restrict__ delta,
                                const float* __restrict__ lse, float* __restrict__ lse2) {
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= rows * nh) return;
  const int64_t row = w / nh;
  const int h = static_cast<int>(w % nh);
  const int H = nh * dh;
  float acc = 0.f;
  for (int d = lane * 2; d < dh; d += 64) {
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(o + row * H + h * dh + d);
    const __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(dout + row * H + h * dh + d);
    acc += __bfloat162float(a.x) * __bfloat162float(c.x) + __bfloat162float(a.y) * __bfloat162float(c.y);
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) {
    const int64_t li = (row / S * nh + h) * S + row % S;
    delta[li] = acc;
    lse2[li] = lse[li] * LOG2E;   // log2-domain LSE for the exp2 of the backward
  }
}

// δ with 16-byte loads: one block per row, each thread 32 consecutive features (4 × 8 bf16) of one head,
// dh/32 threads per head reduced with shuffles (d_h ∈ {64, 128}: 2 or 4 lanes)
__global__ void fa_delta_v8_kernel(int S, int nh, int dh, const bf16* __restrict__ o, const bf16* __restrict__ dout,
                                   float* __restrict__ delta, const float* __restrict__ lse, float* __restrict__ lse2) {
  const int64_t row = blockIdx.x;
  const int H = nh * dh;
  const int64_t base = row * H + static_cast<int64_t>(threadIdx.x) * 32;
  float acc = 0.f;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const uint4 a = *reinterpret_cast<const uint4*>(o + base + v * 8);
    const uint4 c = *reinterpret_cast<const uint4*>(dout + base + v * 8);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 fa = __bfloat1622float2(a2[i]), fc = __bfloat1622float2(c2[i]);
      acc += fa.x * fc.x + fa.y * fc.y;
    }
  }
  const int per_head = dh / 32;
  for (int sft = 1; sft < per_head; sft <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sft);
  if (threadIdx.x % per_head == 0) {
    const int h = threadIdx.x / per_head;
    const int64_t li = (row / S * nh + h) * S + row % S;
    delta[li] = acc;
    lse2[li] = lse[li] * LOG2E;   // log2-domain LSE for the exp2 of the backward
  }
}

// dq (bf16, × softmax scale) <- fp32 accumulator
__global__ void fa_dq_convert_kernel(int64_t rows, int H, const float* __restrict__ acc, bf16* __restrict__ dqkv,
                                     float scale) {
  const int64_t n = rows * H / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(acc)[i];
    const int64_t e = i * 4;
    const int64_t r = e / H, c = e % H;
    uint2 o;
    o.x = pack_bf16(v.x * scale, v.y * scale);
    o.y = pack_bf16(v.z * scale, v.w * scale);
    *reinterpret_cast<uint2*>(dqkv + r * 3 * H + c) = o;
  }
}

// the same conversion fused with the inverse RoPE of dq (rotation by −p·θ_i, p = row mod S): each thread takes
// 4 consecutive columns i..i+3 of the first half of a head and their partners i + d_h/2
__global__ void fa_dq_convert_rope_kernel(int64_t rows, int S, int nh, int dh, const float* __restrict__ acc,
                                          bf16* __restrict__ dqkv, float scale, const float* __restrict__ rcos,
                                          const float* __restrict__ rsin) {
  const int half = dh / 2, H = nh * dh;
  const int64_t per_row = static_cast<int64_t>(nh) * half / 4;
  const int64_t n = rows * per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / per_row;
    const int q = static_cast<int>(i % per_row);
    const int head = q / (half / 4), i0 = (q % (half / 4)) * 4;
    const int64_t base = r * H + static_cast<int64_t>(head) * dh + i0;
    const float4 x1 = *reinterpret_cast<const float4*>(acc + base);
    const float4 x2 = *reinterpret_cast<const float4*>(acc + base + half);
    const int64_t t = (r % S) * half + i0;
    const float4 cc = *reinterpret_cast<const float4*>(rcos + t);
    const float4 ss = *reinterpret_cast<const float4*>(rsin + t);
    const float a[4] = {x1.x * scale, x1.y * scale, x1.z * scale, x1.w * scale};
    const float b[4] = {x2.x * scale, x2.y * scale, x2.z * scale, x2.w * scale};
    const float cv[4] = {cc.x, cc.y, cc.z, cc.w}, sv[4] = {ss.x, ss.y, ss.z, ss.w};
    float y1[4], y2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      y1[k] = a[k] * cv[k] + b[k] * sv[k];
      y2[k] = b[k] * cv[k] - a[k] * sv[k];
    }
    bf16* d = dqkv + r * 3 * H + static_cast<int64_t>(head) * dh + i0;
    *reinterpret_cast<uint2*>(d) = make_uint2(pack_bf16(y1[0], y1[1]), pack_bf16(y1[2], y1[3]));
    *reinterpret_cast<uint2*>(d + half) = make_uint2(pack_bf16(y2[0], y2[1]), pack_bf16(y2[2], y2[3]));
  }
}

// Raise the dynamic shared-memory limit of `kern` once per (kernel, device): the attribute is per device, and a
// process may bootstrap onto another GPU after a finalize.
template <typename K>
void prep(K kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert({reinterpret_cast<const void*>(kern), dev}).second)
    TP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

// TAWPIPE_FA_TRACE=1: per-call clock64 timeline of CTA 0's first 32 key tiles (a tuning aid; allocated and freed
// per call, never on the default path)
struct FaTrace {
  unsigned long long* p = nullptr;
  FaTrace() {
    if (std::getenv("TAWPIPE_FA_TRACE")) {
      TP_CUDA(cudaMalloc(&p, 32 * 16 * 8));
      TP_CUDA(cudaMemset(p, 0, 32 * 16 * 8));
    }
  }
  void dump(const char* const* names, int t0_ev) {
    if (!p) return;
    unsigned long long h[32 * 16];
    TP_CUDA(cudaMemcpy(h, p, sizeof(h), cudaMemcpyDeviceToHost));
    const unsigned long long t0 = h[t0_ev];
    for (int it = 0; it < 12; ++it) {
      std::fprintf(stderr, "it %2d:", it);
      for (int e = 0; e < 16 && names[e]; ++e) std::fprintf(stderr, " %s=%lld", names[e], (long long)(h[it * 16 + e] - t0));
      std::fprintf(stderr, "\n");
    }
  }
  ~FaTrace() {
    if (p) cudaFree(p);
  }
};

}  // namespace

bool attention_tc_supported(int S, int dh) { return S % 128 == 0 && (dh == 64 || dh == 128); }

// Forward: fa_fwd7 (two query tiles per CTA) when the number of query tiles is even, else fa_fwd3.
void attention_fwd_tc(int B, int S, int nh, int dh, const bf16* qkv, bf16* o, float* lse, cudaStream_t s) {
  TP_CHECK(attention_tc_supported(S, dh), TAWPIPE_ECONFIG, "tcgen05 attention: S % 128 == 0, d_h in {64, 128}");
  const int H = nh * dh;
  CUtensorMap tm = make_tmap_bf16_2d(qkv, 3ll * H, static_cast<int64_t>(B) * S, 3ll * H, 128);
  const float scale2 = LOG2E / sqrtf(static_cast<float>(dh));
  if ((S / BQ) % 2 == 0) {
    dim3 grid7(static_cast<unsigned>((S / BQ / 2) * nh), static_cast<unsigned>(B));
    if (dh == 128) {
      prep(fa_fwd7_kernel<128>, Fwd5Smem<128>::BYTES);
      fa_fwd7_kernel<128><<<grid7, 352, Fwd5Smem<128>::BYTES, s>>>(tm, o, lse, S, nh, scale2);
    } else {
      prep(fa_fwd7_kernel<64>, Fwd5Smem<64>::BYTES);
      fa_fwd7_kernel<64><<<grid7, 352, Fwd5Smem<64>::BYTES, s>>>(tm, o, lse, S, nh, scale2);
    }
  } else {
    FaTrace tr;
    dim3 grid3(static_cast<unsigned>((S / BQ) * nh), static_cast<unsigned>(B));
    if (dh == 128) {
      prep(fa_fwd3_kernel<128>, Fwd3Smem<128>::BYTES);
      fa_fwd3_kernel<128><<<grid3, 224, Fwd3Smem<128>::BYTES, s>>>(tm, o, lse, S, nh, scale2, tr.p);
    } else {
      prep(fa_fwd3_kernel<64>, Fwd3Smem<64>::BYTES);
      fa_fwd3_kernel<64><<<grid3, 224, Fwd3Smem<64>::BYTES, s>>>(tm, o, lse, S, nh, scale2, tr.p);
    }
    TP_CUDA(cudaGetLastError());
    static const char* names[16] = {"mma:p_ready", "mma:v_full", "mma:issued", "smx:s_full", "smx:p_done", nullptr};
    tr.dump(names, 3);
  }
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
}

// Backward: δ / log2-domain LSE pre-pass, fa_bwd (dK, dV in TMEM; dQ reduce-added into the fp32 dq_acc), then the
// scaled dQ conversion into dqkv.  scratch: 2·B·n_h·S floats (δ, then LSE·log2e), owned by the caller.
void attention_bwd_tc(int B, int S, int nh, int dh, const bf16* qkv, const bf16* o, const float* lse,
                      const bf16* dout, bf16* dqkv, float* scratch, float* dq_acc, cudaStream_t s, const float* rope_cos,
                      const float* rope_sin) {
  TP_CHECK(attention_tc_supported(S, dh), TAWPIPE_ECONFIG, "tcgen05 attention: S % 128 == 0, d_h in {64, 128}");
  TP_CHECK(dq_acc != nullptr && scratch != nullptr, TAWPIPE_ECONFIG,
           "tcgen05 attention backward needs the δ/LSE scratch and the fp32 dq accumulator");
  const int H = nh * dh;
  const int64_t rows = static_cast<int64_t>(B) * S;
  float* delta = scratch;
  float* lse2 = scratch + rows * nh;
  if (H % 32 == 0 && H / 32 <= 1024 && (dh == 64 || dh == 128))
    fa_delta_v8_kernel<<<static_cast<unsigned>(rows), H / 32, 0, s>>>(S, nh, dh, o, dout, delta, lse, lse2);
  else
    fa_delta_kernel<<<static_cast<unsigned>((rows * nh * 32 + 255) / 256), 256, 0, s>>>(rows, S, nh, dh, o, dout,
                                                                                      delta, lse, lse2);
  TP_CUDA(cudaMemsetAsync(dq_acc, 0, rows * H * sizeof(float), s));
  CUtensorMap tm = make_tmap_bf16_2d(qkv, 3ll * H, rows, 3ll * H, 128);
  CUtensorMap tmdo = make_tmap_bf16_2d(dout, H, rows, H, 128);
  CUtensorMap tmdq = make_tmap_f32_2d(dq_acc, H, rows, H, 128);
  const float scale = 1.0f / sqrtf(static_cast<float>(dh));
  const float scale2 = LOG2E * scale;
  dim3 grid(static_cast<unsigned>((S / BQ) * nh), static_cast<unsigned>(B));
  FaTrace tr;
  if (dh == 128) {
    prep(fa_bwd_kernel<128>, BwdSmem<128>::BYTES);
    fa_bwd_kernel<128><<<grid, 352, BwdSmem<128>::BYTES, s>>>(tm, tmdo, tmdq, lse2, delta, dq_acc, dqkv, S, nh, scale,
                                                               scale2, tr.p, rope_cos, rope_sin);
  } else {
    prep(fa_bwd_kernel<64>, BwdSmem<64>::BYTES);
    fa_bwd_kernel<64><<<grid, 352, BwdSmem<64>::BYTES, s>>>(tm, tmdo, tmdq, lse2, delta, dq_acc, dqkv, S, nh, scale,
                                                             scale2, tr.p, rope_cos, rope_sin);
  }
  TP_CUDA(cudaGetLastError());
  if (rope_cos)
    fa_dq_convert_rope_kernel<<<148 * 8, 256, 0, s>>>(rows, S, nh, dh, dq_acc, dqkv, scale, rope_cos, rope_sin);
  else
    fa_dq_convert_kernel<<<148 * 8, 256, 0, s>>>(rows, H, dq_acc, dqkv, scale);
  TP_CUDA(cudaGetLastError());
  static const char* names[16] = {"mma:S_issued", "mma:dO+tdp_free", "mma:p_ready", "mma:ds_ready", "cmp:s_full",
                                  "cmp:p_done", "cmp:dp_full", "cmp:mm2_prev", "cmp:ds_done", "dq:mm2_done",
                                  "dq:tdp_free", "dq:staged", "cmp:ds_w0", "cmp:ds_w1", "cmp:ds_w2", "cmp:ds_w3"};
  tr.dump(names, 0);
  g_kstats.launches += 3;
}

}  // namespace tp
