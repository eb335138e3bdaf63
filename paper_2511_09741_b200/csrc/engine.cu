// engine.cu -- DBS plan, GWPS/CCO step engine and the C ABI of libtawpipe.
//
// Paper mapping (§3; readings R1-R21 in SURVEY.md §8(c), listed in DESIGN.md):
//   DBS      : layer l is owned by group l mod D, striped over its G members (R6); each rank keeps
//                             fp32 master / m / v and a wire-dtype copy of its owned stripes only.
//   GWPS : per layer, rail P2P of stripe j from the owner group (inter-group, "wp"), then an
//                             intra-group all-gather ("wb"); gradients are reduce-scattered in the group ("gr")
//                             and sent on the rail to the owner ("gp"), which sums the D group contributions in
//                             ascending group order and applies AdamW locally (R16).
//   CCO : gathers run on a weight stream (ws) one layer ahead of the compute stream (cs),
//                             into double-buffered layer slots; gradient reduction + AdamW run on a third stream (gs).
// Every step of the path runs in this library's kernels; torch only bootstraps the process group (no CPU fallback).
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "common.cuh"
#include "peer.cuh"

namespace tp {

#define TP_NCCL(x)                                                                                             \
  do {                                                                                                         \
    ncclResult_t r_ = (x);                                                                                     \
    if (r_ != ncclSuccess)                                                                                     \
      throw ::tp::Error(TAWPIPE_ERUNTIME, std::string("NCCL: ") + ncclGetErrorString(r_) + " at " + __FILE__ + \
                                              ":" + std::to_string(__LINE__));                                 \
  } while (0)

namespace {

enum { U_BLOCK = 0, U_E = 1, U_F = 2 };
enum { K_W = 0, K_G = 1 };
enum { C_INTRA = 0, C_INTER = 1 };
enum { D_RECV = 0, D_SENT = 1 };
inline int ledger_index(int kind, int cls, int dir, int unit) { return ((kind * 2 + cls) * 2 + dir) * 3 + unit; }

struct Unit {
  int cls = U_BLOCK;
  int64_t n = 0, n_pad = 0, s = 0;  // elements, padded, stripe
  int owner = 0;                    // owner group
  bool owned = false;
  int64_t off = 0;                  // offset of this rank's stripe in the owned-state arrays
  int64_t canon = 0;                // offset of the unit in the canonical full-model vector
  int64_t lo = 0;                   // unit coordinate of this rank's owned piece (striped: j·s; whole units: 0)
  int hold = 0;                     // TAWPIPE_LITERAL: member index of the owner inside its group and of the
                                    // holder / staging / exit device inside every group (rail counterpart, R7)
  int n_nd = 0;
  int64_t nd_lo[2] = {0, 0}, nd_hi[2] = {0, 0};  // no-decay ranges (unit coordinates)
};

struct Acts {  // one (layer, micro-batch) forward's saved tensors
  void *a, *qkv, *o, *h1, *b, *gu, *y;
  float *r1, *lse, *r2;
};

// Selective checkpointing (ckpt = 1): beyond the residual checkpoint h_l, the step keeps, for as many
// (layer, micro-batch) pairs as the device memory left after everything else allows, in this order:
//   KEEP_ATTN  attention output O and LSE       (recompute skips the attention forward)
//   KEEP_QKV   post-RoPE q|k|v                   (skips the QKV GEMM and RoPE)
//   KEEP_H1    h1 = h + O·Woᵀ                    (skips the O GEMM)
//   KEEP_MLP   gu = [x·Wgateᵀ | x·Wupᵀ]            (skips the gate/up GEMM; y = SwiGLU(gu) is re-derived by the
//                                                 elementwise kernel: 1.4 GB kept per layer instead of 2.2)
// The two RMSNorms are always recomputed (cheap; their outputs and 1/rms feed the backward).  A kept tensor is
// the output of the same kernel on the same inputs as its recompute would be, so results are bit-identical, except
// y at the MLP level: re-derived from the bf16 gu rather than the GEMM epilogue's fp32 accumulators (one bf16
// rounding apart).
enum : uint8_t { KEEP_ATTN = 1, KEEP_QKV = 2, KEEP_H1 = 4, KEEP_MLP = 8 };
struct Kept {
  uint8_t flags = 0;
  void *o = nullptr, *qkv = nullptr, *h1 = nullptr, *gu = nullptr;
  float* lse = nullptr;
};

struct TimedRegion {
  cudaEvent_t a, b;
  int kind;  // 0 gemm, 1 attention, 2 adamw, 3 exposed wait, 4 elementwise, 5 weight comm, 6 grad comm
  double work;
  int stream;  // 0 compute, 1 weights, 2 gradients
};

struct Ctx {
  // process / topology
  int rank = 0, world = 1, device = 0;
  bool booted = false, inited = false;
  ncclComm_t world_comm = nullptr;
  int P = 1, G = 1, D = 1, k = 0, j = 0, L = 0, N = 1, m = 1;
  tawpipe_dims dims{};
  int H = 0, nh = 0, dh = 0, I = 0, V = 0, S = 0, Bm = 1;
  int64_t T = 0, phi = 0;
  bool bf = false;
  bool ring = false;     // TAWPIPE_RING schedule
  bool literal = false;  // TAWPIPE_LITERAL: whole-layer owners, broadcast / reduce in the group (NEXT-2)
  size_t esz = 4;
  ncclComm_t wg = nullptr, wr = nullptr, gg = nullptr, gr = nullptr;
  cudaStream_t cs = nullptr, ws = nullptr, gs = nullptr;
  std::vector<Unit> units;  // 0..L-1 layers, L = E, L+1 = F
  int64_t owned_total = 0, max_pad = 0, max_s = 0;
  float *master = nullptr, *mom = nullptr, *vel = nullptr;
  void* wire = nullptr;
  void* wbuf[2] = {nullptr, nullptr};
  void *ebuf = nullptr, *fbuf = nullptr;
  float* gacc[2] = {nullptr, nullptr};
  float *gaccE = nullptr, *gaccF = nullptr;
  void *gwire = nullptr, *rsout = nullptr, *crecv = nullptr;
  // activations
  std::vector<void*> ck;  // (L+1) * m  residual-stream checkpoints h_l
  std::vector<Acts> acts;  // L*m (no ckpt) or 1 (ckpt)
  std::vector<Kept> kept;  // L*m under ckpt == 1: activations kept beyond h_l (memory-budgeted)
  double recompute_gflop = 0;  // algorithmic work of the recompute passes of the last step
  std::string trace_json;      // Trace-Event JSON of the last timed step (NEXT-4)
  // emulated link hierarchy (NEXT-3): transfers that cross an emulated node boundary are paced
  double emu_gbps = 0, emu_lat_us = 0;
  int emu_node = 0;            // devices per emulated node (0: the schedule's group size G)
  std::vector<void*> dhb;  // m: gradient of the residual stream per micro-batch
  void *dY = nullptr, *dGU = nullptr, *db = nullptr, *dh1 = nullptr, *dO = nullptr, *dqkv = nullptr, *da = nullptr;
  float *delta = nullptr, *dq_acc = nullptr;
  void* barrier_buf = nullptr;  // one int for world_barrier
  void* emb_scratch = nullptr;  // deterministic embedding backward: sort keys / positions + CUB temp
  size_t emb_scratch_bytes = 0;
  void *fnorm = nullptr, *logits = nullptr, *df = nullptr;
  float *rstd_f = nullptr, *loss_rows = nullptr;
  int64_t Tc = 0;
  int32_t *d_tok = nullptr, *d_in = nullptr, *d_tgt = nullptr, *h_tok = nullptr;
  float *cosT = nullptr, *sinT = nullptr;
  float* rope_cs = nullptr;   // [S][d_h]: cos | sin per position, for the RoPE epilogue of the QKV GEMM (bf16 path)
  double* d_loss = nullptr;
  double* h_loss = nullptr;
  uint64_t ledger[TAWPIPE_LEDGER_N] = {};
  uint64_t ledger_plan[TAWPIPE_LEDGER_N] = {};   // what the documented schedule moves per step (plan_ledger)
  float* dg_scratch = nullptr;   // RMSNorm dγ row-block partials (rmsnorm_bwd_scratch_floats(T, H))
  int step_t = 0;
  // NVLink peer path of the GWPS schedule (peer.cu): IPC-mapped buffers of every rank, sequence flags
  bool p2p = false;
  std::vector<std::vector<void*>> peer;   // [rank][PB_*]
  std::vector<int64_t> gofs;              // [group][unit]: offset of the unit's stripe in that group's owned arrays
  uint32_t* sig = nullptr;                // this rank's flags [SK_*][source rank]
  void* part = nullptr;                   // rail partials of this rank's group (4 slots: layer 0/1, E, F) × max_s
  uint32_t wseq = 0, gseq = 0;            // gathers / reductions issued so far (identical on every rank)
  int slot_tag[2][2] = {{-1, -1}, {-1, -1}};   // [slot] = {unit, step} of the last gather into it
  uint32_t wprev[2] = {0, 0}, gprev[2] = {0, 0}, pprev[4] = {0, 0, 0, 0};
  int pprev_owner[4] = {0, 0, 0, 0};      // the rank that read the previous partial in that slot
  double nvl_w_bytes = 0, nvl_g_bytes = 0;   // bytes this rank pulled / read over NVLink in the last step
  std::vector<uint32_t> sig_expect;       // [SK_* · kSigRanks + src]: the last value each peer must have written
  // events
  cudaEvent_t w_ready[2], w_free[2], g_ready[2], g_free[2], evE, evF, evGF, evGE, ev_s0, ev_s1, ev_ws0, ev_ws1,
      ev_gs0, ev_gs1;
  // timing
  bool timing = false;
  std::vector<TimedRegion> regions;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  double stats[TAWPIPE_STATS_N] = {};
  size_t bytes_alloc = 0;
  std::vector<void*> allocs;
  long launches_at_start = 0;
};

// peer buffers (Ctx::peer[rank][PB_*]) and signal kinds (Ctx::sig[SK_* · kSigRanks + source rank])
enum { PB_WIRE, PB_WBUF0, PB_WBUF1, PB_EBUF, PB_FBUF, PB_GACC0, PB_GACC1, PB_GACCE, PB_GACCF, PB_PART, PB_SIG, PB_N };
enum { SK_RAIL, SK_WDONE, SK_GREADY, SK_GDONE, SK_PREADY, SK_PDONE, SK_N };
constexpr int kSigRanks = 64;

Ctx* g = nullptr;
thread_local std::string g_err = "no error";
}  // namespace
void set_last_error(const std::string& msg) { g_err = msg; }
namespace {

void* dmalloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 256;
  TP_CUDA(cudaMalloc(&p, bytes));
  g->allocs.push_back(p);
  g->bytes_alloc += bytes;
  return p;
}

// Device-side barrier of all ranks (a one-int NCCL all-reduce on the compute stream, then a host wait).  The
// peer path pulls owners' wire copies without a rendezvous, so every operation that rewrites them outside a step
// (the device-side init in tawpipe_init, tawpipe_load) ends with this barrier.
void world_barrier() {
  if (g->world <= 1) return;
  int* d = static_cast<int*>(g->barrier_buf);
  TP_NCCL(ncclAllReduce(d, d, 1, ncclInt, ncclSum, g->world_comm, g->cs));
  TP_CUDA(cudaStreamSynchronize(g->cs));
}

cudaEvent_t pool_event() {
  if (g->ev_used == g->ev_pool.size()) {
    cudaEvent_t e;
    TP_CUDA(cudaEventCreate(&e));
    g->ev_pool.push_back(e);
  }
  return g->ev_pool[g->ev_used++];
}

bool trace_on() {
  static const bool on = std::getenv("TAWPIPE_TRACE") != nullptr;
  return on;
}
#define TRACE(...)                                 \
  do {                                             \
    if (trace_on()) {                              \
      std::fprintf(stderr, "[tawpipe] " __VA_ARGS__); \
      std::fflush(stderr);                         \
    }                                              \
  } while (0)

struct Timed {  // RAII CUDA-event bracket on a stream (only when timing is enabled)
  cudaStream_t s;
  TimedRegion r{};
  bool on;
  Timed(cudaStream_t st, int kind, double work) : s(st), on(g->timing) {
    if (trace_on()) {
      TP_CUDA(cudaDeviceSynchronize());
      TRACE("region kind %d work %.3g start\n", kind, work);
    }
    if (!on) return;
    r.a = pool_event();
    r.b = pool_event();
    r.kind = kind;
    r.work = work;
    r.stream = st == g->cs ? 0 : st == g->ws ? 1 : 2;
    TP_CUDA(cudaEventRecord(r.a, s));
  }
  // never throws: a destructor that runs while an exception unwinds must not raise a second one (that would
  // terminate the process instead of returning TAWPIPE_ERUNTIME); a failed record is kept in g_err and the
  // region is dropped
  ~Timed() noexcept {
    if (trace_on()) {
      const cudaError_t e = cudaDeviceSynchronize();
      TRACE("region kind %d done (%s)\n", r.kind, cudaGetErrorString(e));
    }
    if (!on || std::uncaught_exceptions() > 0) return;
    const cudaError_t e = cudaEventRecord(r.b, s);
    if (e != cudaSuccess) {
      g_err = std::string("CUDA: ") + cudaGetErrorString(e) + " recording a timing event";
      return;
    }
    g->regions.push_back(r);
  }
};

inline ncclDataType_t wire_type() { return g->bf ? ncclBfloat16 : ncclFloat32; }
inline char* wptr(void* base, int64_t elems) { return static_cast<char*>(base) + elems * static_cast<int64_t>(g->esz); }

// ------------------------------------------------------------------------------------ link emulation (NEXT-3)
// With tawpipe_set_link_emulation on, a transfer whose endpoints lie in different emulated nodes (node of device d
// = d / node_size) is followed, on every participating stream, by a device-side delay of latency + bytes / bandwidth,
// where bytes is what the busiest endpoint moves across the node boundary in that exchange (alpha-beta model,
// SPEC.md:85 "a800-10gbe": 1.25 GB/s, 30 µs).  The data and the ledger are unchanged; only time is added.
int emu_node_size() { return g->emu_node > 0 ? g->emu_node : g->G; }
bool emu_crosses(int a, int b) { return g->emu_gbps > 0 && a / emu_node_size() != b / emu_node_size(); }
void emu_delay(double bytes, cudaStream_t s) {
  if (g->emu_gbps <= 0) return;
  link_delay(g->emu_lat_us * 1e-6 + bytes / (g->emu_gbps * 1e9), s);
}
// rail exchange among the D devices (kk·G + j): crosses nodes iff the rail spans more than one emulated node
bool emu_rail_crosses() { return g->D > 1 && emu_crosses(g->j, (g->D - 1) * g->G + g->j); }
// group collective among devices k·G .. k·G + G − 1
bool emu_group_crosses() { return g->G > 1 && emu_crosses(g->k * g->G, g->k * g->G + g->G - 1); }

// ------------------------------------------------------------------------------------ kernel dispatch
bool gemm_force_simt() {
  static const bool force_simt = [] {
    const char* e = std::getenv("TAWPIPE_GEMM");
    return e && std::string(e) == "simt";
  }();
  return force_simt;
}

void gemm(int64_t M, int64_t Nn, int64_t K, const void* A, int64_t lda, bool akm, const void* B, int64_t ldb, bool bkm,
          void* C, int64_t ldc, bool c_f32, bool acc, const void* R, cudaStream_t s) {
  GemmArgs a{M, Nn, K, A, lda, akm, B, ldb, bkm, C, ldc, c_f32, acc, R};
  Timed t(s, 0, 2.0 * M * Nn * K);
  if (!g->bf)
    gemm_simt<float>(a, s);
  else if (gemm_force_simt())
    gemm_simt<bf16>(a, s);
  else
    gemm_tc_bf16(a, s);
}

bool use_tc_attention() {
  static const int mode = [] {
    const char* e = std::getenv("TAWPIPE_ATTN");
    if (e && std::string(e) == "simt") return 0;
    return 1;
  }();
  return g->bf && mode == 1 && attention_tc_supported(g->S, g->dh);
}

double attn_flops_fwd() {  // causal: QKᵀ and PV each H·S(S+1) MACs per sequence -> 2·2·H·S(S+1)/2·... (App. B)
  return 2.0 * g->H * (g->S + 1.0) * g->S * g->Bm;
}

void attn_fwd(const void* qkv, void* o, float* lse, cudaStream_t s) {
  Timed t(s, 1, attn_flops_fwd());
  if (!g->bf)
    attention_fwd_simt<float>(g->Bm, g->S, g->nh, g->dh, (const float*)qkv, (float*)o, lse, s);
  else if (use_tc_attention())
    attention_fwd_tc(g->Bm, g->S, g->nh, g->dh, (const bf16*)qkv, (bf16*)o, lse, s);
  else
    attention_fwd_simt<bf16>(g->Bm, g->S, g->nh, g->dh, (const bf16*)qkv, (bf16*)o, lse, s);
}
void attn_bwd(const void* qkv, const void* o, const float* lse, const void* dout, void* dqkv, cudaStream_t s) {
  Timed t(s, 1, 2.0 * attn_flops_fwd());
  if (!g->bf)
    attention_bwd_simt<float>(g->Bm, g->S, g->nh, g->dh, (const float*)qkv, (const float*)o, lse, (const float*)dout,
                              (float*)dqkv, g->delta, s);
  else if (use_tc_attention())   // the inverse RoPE of dq / dk is fused into the kernel's dq and dK outputs
    attention_bwd_tc(g->Bm, g->S, g->nh, g->dh, (const bf16*)qkv, (const bf16*)o, lse, (const bf16*)dout,
                     (bf16*)dqkv, g->delta, g->dq_acc, s, g->cosT, g->sinT);
  else
    attention_bwd_simt<bf16>(g->Bm, g->S, g->nh, g->dh, (const bf16*)qkv, (const bf16*)o, lse, (const bf16*)dout,
                             (bf16*)dqkv, g->delta, s);
}

#define BY_TYPE(call_f32, call_bf16) \
  do {                               \
    if (g->bf) {                     \
      call_bf16;                     \
    } else {                         \
      call_f32;                      \
    }                                \
  } while (0)

void k_rmsnorm_fwd(const void* x, const void* gm, void* y, float* r, int64_t rows, cudaStream_t s) {
  Timed t(s, 4, 0);
  BY_TYPE(rmsnorm_fwd<float>((const float*)x, (const float*)gm, (float*)y, r, rows, g->H, g->dims.rms_eps, s),
          rmsnorm_fwd<bf16>((const bf16*)x, (const bf16*)gm, (bf16*)y, r, rows, g->H, g->dims.rms_eps, s));
}
void k_rmsnorm_bwd(const void* dy, const void* x, const void* gm, const float* r, const void* res, void* dx,
                   float* dgacc, int64_t rows, cudaStream_t s) {
  Timed t(s, 4, 0);
  BY_TYPE(rmsnorm_bwd<float>((const float*)dy, (const float*)x, (const float*)gm, r, (const float*)res, (float*)dx,
                             dgacc, g->dg_scratch, rows, g->H, s),
          rmsnorm_bwd<bf16>((const bf16*)dy, (const bf16*)x, (const bf16*)gm, r, (const bf16*)res, (bf16*)dx, dgacc,
                            g->dg_scratch, rows, g->H, s));
}
void k_rope(void* qkv, bool inverse, cudaStream_t s) {
  Timed t(s, 4, 0);
  BY_TYPE(rope_apply<float>((float*)qkv, g->Bm, g->S, g->nh, g->dh, g->cosT, g->sinT, inverse, 2, s),
          rope_apply<bf16>((bf16*)qkv, g->Bm, g->S, g->nh, g->dh, g->cosT, g->sinT, inverse, 2, s));
}

// ------------------------------------------------------------------------------------ comm (a3, a8)
// Logical-element ledger of one gather / one reduction of unit u on device (k, j):
// all-gather and reduce-scatter: (G-1)·s received and sent per participant; P2P: s per message.
void ledger_gather(const Unit& u, int G, int D, uint64_t* led) {
  if (D > 1) {
    if (u.owned)
      led[ledger_index(K_W, C_INTER, D_SENT, u.cls)] += static_cast<uint64_t>(u.s) * (D - 1);
    else
      led[ledger_index(K_W, C_INTER, D_RECV, u.cls)] += static_cast<uint64_t>(u.s);
  }
  if (G > 1) {
    led[ledger_index(K_W, C_INTRA, D_RECV, u.cls)] += static_cast<uint64_t>(u.s) * (G - 1);
    led[ledger_index(K_W, C_INTRA, D_SENT, u.cls)] += static_cast<uint64_t>(u.s) * (G - 1);
  }
}
// WeiPipe-style ring (G = 1): device d receives layer u from d-1 unless it owns it and forwards it to d+1
// unless d+1 owns it; the gradient partial starts at owner+1 and ends at the owner (one P2P per hop).
void ledger_gather_ring(const Unit& u, int d, int P, uint64_t* led) {
  if (P == 1) return;
  if (d != u.owner) led[ledger_index(K_W, C_INTER, D_RECV, u.cls)] += static_cast<uint64_t>(u.s);
  if ((d + 1) % P != u.owner) led[ledger_index(K_W, C_INTER, D_SENT, u.cls)] += static_cast<uint64_t>(u.s);
}
void ledger_reduce_ring(const Unit& u, int d, int P, uint64_t* led) {
  if (P == 1) return;
  if (d != (u.owner + 1) % P) led[ledger_index(K_G, C_INTER, D_RECV, u.cls)] += static_cast<uint64_t>(u.s);
  if (d != u.owner) led[ledger_index(K_G, C_INTER, D_SENT, u.cls)] += static_cast<uint64_t>(u.s);
}
// TAWPIPE_LITERAL (NEXT-2): whole units, owner (k_o, i), holder (k, i) in every group k.  Gather: rail P2P owner ->
// (k, i) for k != k_o, then broadcast from (k, i) in each group.  Reduction: reduce to (k, i) in each group, then
// rail P2P (k, i) -> owner for k != k_o.  Broadcast of x: each non-root receives x, the root sends (G−1)·x
// (reading R23 of SURVEY App. A's "—"); reduce of x: the root receives (G−1)·x, each non-root sends x.
void ledger_gather_literal(const Unit& u, int G, int D, int k, int j, uint64_t* led) {
  const uint64_t x = static_cast<uint64_t>(u.n_pad);
  if (D > 1 && j == u.hold) {
    if (k == u.owner) led[ledger_index(K_W, C_INTER, D_SENT, u.cls)] += x * (D - 1);
    else led[ledger_index(K_W, C_INTER, D_RECV, u.cls)] += x;
  }
  if (G > 1) {
    if (j == u.hold) led[ledger_index(K_W, C_INTRA, D_SENT, u.cls)] += x * (G - 1);
    else led[ledger_index(K_W, C_INTRA, D_RECV, u.cls)] += x;
  }
}
void ledger_reduce_literal(const Unit& u, int G, int D, int k, int j, uint64_t* led) {
  const uint64_t x = static_cast<uint64_t>(u.n_pad);
  if (G > 1) {
    if (j == u.hold) led[ledger_index(K_G, C_INTRA, D_RECV, u.cls)] += x * (G - 1);
    else led[ledger_index(K_G, C_INTRA, D_SENT, u.cls)] += x;
  }
  if (D > 1 && j == u.hold) {
    if (k == u.owner) led[ledger_index(K_G, C_INTER, D_RECV, u.cls)] += x * (D - 1);
    else led[ledger_index(K_G, C_INTER, D_SENT, u.cls)] += x;
  }
}

void ledger_reduce(const Unit& u, int G, int D, uint64_t* led) {
  if (G > 1) {
    led[ledger_index(K_G, C_INTRA, D_RECV, u.cls)] += static_cast<uint64_t>(u.s) * (G - 1);
    led[ledger_index(K_G, C_INTRA, D_SENT, u.cls)] += static_cast<uint64_t>(u.s) * (G - 1);
  }
  if (D > 1) {
    if (u.owned)
      led[ledger_index(K_G, C_INTER, D_RECV, u.cls)] += static_cast<uint64_t>(u.s) * (D - 1);
    else
      led[ledger_index(K_G, C_INTER, D_SENT, u.cls)] += static_cast<uint64_t>(u.s);
  }
}

// full unit buffer the compute reads for unit u (slot for layers)
void* unit_buffer(int uid, int slot) {
  const Unit& u = g->units[uid];
  if (g->G == 1 && u.owned) return wptr(g->wire, u.off);
  if (u.cls == U_E) return g->ebuf;
  if (u.cls == U_F) return g->fbuf;
  return g->wbuf[slot];
}

void gather_p2p(int uid, int slot);
void reduce_p2p(int uid, int slot, float* gacc);

// a3: rail P2P of stripe j from the owner group (if remote) + intra-group all-gather, on ws
// Version tags of the two layer slots (SURVEY §8(b) "version tag" invariant): the unit and step the last gather into
// each slot was issued for; the compute checks them before reading a slot (host-side, every step).
void tag_slot(int uid, int slot) {
  if (g->units[uid].cls != U_BLOCK) return;
  g->slot_tag[slot][0] = uid;
  g->slot_tag[slot][1] = g->step_t;
}
void check_slot(int uid, int slot) {
  const Unit& u = g->units[uid];
  if (g->P == 1 || (g->G == 1 && u.owned)) return;   // the compute reads the owned wire copy, not a slot
  if (g->slot_tag[slot][0] != uid || g->slot_tag[slot][1] != g->step_t)
    throw Error(TAWPIPE_EINVARIANT, "layer slot " + std::to_string(slot) + " holds unit " +
                                        std::to_string(g->slot_tag[slot][0]) + " of step " +
                                        std::to_string(g->slot_tag[slot][1]) + ", compute needs layer " +
                                        std::to_string(uid) + " of step " + std::to_string(g->step_t));
}

void gather(int uid, int slot) {
  const Unit& u = g->units[uid];
  tag_slot(uid, slot);
  if (g->P == 1) return;  // nothing to move; the compute reads the owned copy in place
  if (g->p2p) {
    gather_p2p(uid, slot);
    return;
  }
  void* dst = unit_buffer(uid, slot);
  Timed t(g->ws, 5, 0);
  void* own = wptr(g->wire, u.off);
  if (g->ring) {  // owner -> owner+1 -> ... : receive from d-1, then forward to d+1 (stream-ordered)
    const int d = g->rank, P = g->P;
    void* buf = u.owned ? own : dst;
    if (!u.owned) {
      TP_NCCL(ncclRecv(buf, u.n_pad, wire_type(), (d + P - 1) % P, g->wr, g->ws));
      if (emu_crosses((d + P - 1) % P, d)) emu_delay(static_cast<double>(u.n_pad) * g->esz, g->ws);
    }
    if ((d + 1) % P != u.owner) {
      TP_NCCL(ncclSend(buf, u.n_pad, wire_type(), (d + 1) % P, g->wr, g->ws));
      if (emu_crosses(d, (d + 1) % P)) emu_delay(static_cast<double>(u.n_pad) * g->esz, g->ws);
    }
    ledger_gather_ring(u, d, P, g->ledger);
    return;
  }
  if (g->literal) {  // NEXT-2: owner -> rail counterparts, then broadcast from the holder in every group
    const bool holder = (g->j == u.hold);
    if (g->D > 1 && holder) {
      TP_NCCL(ncclGroupStart());
      if (u.owned) {
        for (int kk = 0; kk < g->D; ++kk)
          if (kk != g->k) TP_NCCL(ncclSend(own, u.n_pad, wire_type(), kk, g->wr, g->ws));
      } else {
        TP_NCCL(ncclRecv(dst, u.n_pad, wire_type(), u.owner, g->wr, g->ws));
      }
      TP_NCCL(ncclGroupEnd());
      if (emu_rail_crosses()) emu_delay(static_cast<double>(g->D - 1) * u.n_pad * g->esz, g->ws);
    }
    if (g->G > 1) {
      TP_NCCL(ncclBroadcast(u.owned ? own : dst, dst, u.n_pad, wire_type(), u.hold, g->wg, g->ws));
      if (emu_group_crosses()) emu_delay(static_cast<double>(g->G - 1) * u.n_pad * g->esz, g->ws);
    }
    ledger_gather_literal(u, g->G, g->D, g->k, g->j, g->ledger);
    return;
  }
  if (g->D > 1) {
    TP_NCCL(ncclGroupStart());
    if (u.owned) {
      for (int kk = 0; kk < g->D; ++kk)
        if (kk != g->k) TP_NCCL(ncclSend(own, u.s, wire_type(), kk, g->wr, g->ws));
    } else {
      TP_NCCL(ncclRecv(wptr(dst, g->j * u.s), u.s, wire_type(), u.owner, g->wr, g->ws));
    }
    TP_NCCL(ncclGroupEnd());
    // the owner's link carries its stripe to each of the D − 1 other groups
    if (emu_rail_crosses()) emu_delay(static_cast<double>(g->D - 1) * u.s * g->esz, g->ws);
  }
  if (g->G > 1) {
    const void* send = u.owned ? own : wptr(dst, g->j * u.s);
    TP_NCCL(ncclAllGather(send, dst, u.s, wire_type(), g->wg, g->ws));
    // ring all-gather: each link across the node boundary carries G − 1 stripes
    if (emu_group_crosses()) emu_delay(static_cast<double>(g->G - 1) * u.s * g->esz, g->ws);
  }
  ledger_gather(u, g->G, g->D, g->ledger);
}

// a8 + a9: reduce-scatter in the group, rail P2P to the owner, ascending-k accumulate + AdamW, on gs
void adam_update(const Unit& u, const void* const* contrib, int n_contrib, int own_k, bool own_f32);
void adam_apply(const Unit& u, const GradSources& src, int n_src);

// WeiPipe-style ring reduction: owner+1 starts the partial sum, each device adds its local fp32 gradient and
// forwards it (wire dtype), the owner adds its own and applies AdamW
void reduce_ring(const Unit& u, float* gacc) {
  cudaStream_t s = g->gs;
  const int d = g->rank, P = g->P;
  if (P == 1) {
    const void* c0 = gacc;
    adam_update(u, &c0, 1, 0, true);
    return;
  }
  const int prev = (d + P - 1) % P, next = (d + 1) % P;
  const bool first = (d == (u.owner + 1) % P);
  if (!first) {
    Timed t(s, 6, 0);
    TP_NCCL(ncclRecv(g->crecv, u.n_pad, wire_type(), prev, g->gr, s));
    if (emu_crosses(prev, d)) emu_delay(static_cast<double>(u.n_pad) * g->esz, s);
  }
  if (u.owned) {
    const void* contrib[2] = {gacc, g->crecv};
    adam_update(u, contrib, 2, 0, true);
  } else {
    {
      Timed t(s, 4, 0);
      if (first)
        BY_TYPE(cast_f32<float>(gacc, (float*)g->gwire, u.n_pad, s), cast_f32<bf16>(gacc, (bf16*)g->gwire, u.n_pad, s));
      else
        BY_TYPE(add_cast<float>((const float*)g->crecv, gacc, (float*)g->gwire, u.n_pad, s),
                add_cast<bf16>((const bf16*)g->crecv, gacc, (bf16*)g->gwire, u.n_pad, s));
    }
    Timed t(s, 6, 0);
    TP_NCCL(ncclSend(g->gwire, u.n_pad, wire_type(), next, g->gr, s));
    if (emu_crosses(d, next)) emu_delay(static_cast<double>(u.n_pad) * g->esz, s);
  }
  ledger_reduce_ring(u, d, P, g->ledger);
}

void reduce_and_update(int uid, int slot, float* gacc) {
  const Unit& u = g->units[uid];
  if (g->p2p) {
    reduce_p2p(uid, slot, gacc);
    return;
  }
  if (g->ring) {
    reduce_ring(u, gacc);
    return;
  }
  cudaStream_t s = g->gs;
  if (g->literal) {  // NEXT-2: reduce to the holder in every group, holder -> owner on the rail, owner updates
    const bool holder = (g->j == u.hold);
    const void* partial = gacc;
    bool part_f32 = true;
    if (g->G > 1 || (g->D > 1 && !u.owned)) {
      Timed t(s, 4, 0);
      BY_TYPE(cast_f32<float>(gacc, (float*)g->gwire, u.n_pad, s), cast_f32<bf16>(gacc, (bf16*)g->gwire, u.n_pad, s));
      partial = g->gwire;
      part_f32 = false;
    }
    if (g->G > 1) {
      Timed t(s, 6, 0);
      TP_NCCL(ncclReduce(g->gwire, g->rsout, u.n_pad, wire_type(), ncclSum, u.hold, g->gg, s));
      if (emu_group_crosses()) emu_delay(static_cast<double>(g->G - 1) * u.n_pad * g->esz, s);
      partial = g->rsout;
    }
    if (g->D > 1 && holder) {
      Timed t(s, 6, 0);
      TP_NCCL(ncclGroupStart());
      if (u.owned) {
        int idx = 0;
        for (int kk = 0; kk < g->D; ++kk)
          if (kk != g->k) TP_NCCL(ncclRecv(wptr(g->crecv, (idx++) * u.n_pad), u.n_pad, wire_type(), kk, g->gr, s));
      } else {
        TP_NCCL(ncclSend(partial, u.n_pad, wire_type(), u.owner, g->gr, s));
      }
      TP_NCCL(ncclGroupEnd());
      if (emu_rail_crosses()) emu_delay(static_cast<double>(g->D - 1) * u.n_pad * g->esz, s);
    }
    ledger_reduce_literal(u, g->G, g->D, g->k, g->j, g->ledger);
    if (!u.owned) return;
    const void* contrib[8];
    int idx = 0;
    for (int kk = 0; kk < g->D; ++kk) contrib[kk] = (kk == g->k) ? partial : wptr(g->crecv, (idx++) * u.n_pad);
    adam_update(u, contrib, g->D, g->k, part_f32);
    return;
  }
  const void* own_partial = gacc;
  bool own_f32 = true;
  if (g->G > 1 || (g->D > 1 && !u.owned)) {
    Timed t(s, 4, 0);
    BY_TYPE(cast_f32<float>(gacc, (float*)g->gwire, u.n_pad, s), cast_f32<bf16>(gacc, (bf16*)g->gwire, u.n_pad, s));
    own_partial = g->gwire;
    own_f32 = false;
  }
  if (g->G > 1) {
    Timed t(s, 6, 0);
    TP_NCCL(ncclReduceScatter(g->gwire, g->rsout, u.s, wire_type(), ncclSum, g->gg, s));
    if (emu_group_crosses()) emu_delay(static_cast<double>(g->G - 1) * u.s * g->esz, s);
    own_partial = g->rsout;
  }
  if (g->D > 1) {
    Timed t(s, 6, 0);
    TP_NCCL(ncclGroupStart());
    if (u.owned) {
      int idx = 0;
      for (int kk = 0; kk < g->D; ++kk)
        if (kk != g->k) TP_NCCL(ncclRecv(wptr(g->crecv, (idx++) * u.s), u.s, wire_type(), kk, g->gr, s));
    } else {
      TP_NCCL(ncclSend(own_partial, u.s, wire_type(), u.owner, g->gr, s));
    }
    TP_NCCL(ncclGroupEnd());
    // the owner's link receives the D − 1 group partials
    if (emu_rail_crosses()) emu_delay(static_cast<double>(g->D - 1) * u.s * g->esz, s);
  }
  ledger_reduce(u, g->G, g->D, g->ledger);
  if (!u.owned) return;
  const void* contrib[8];
  int idx = 0;
  for (int kk = 0; kk < g->D; ++kk) contrib[kk] = (kk == g->k) ? own_partial : wptr(g->crecv, (idx++) * u.s);
  adam_update(u, contrib, g->D, g->k, own_f32);
}

// a9: fused accumulate of the group contributions (ascending order) + AdamW on this rank's owned stripe, on gs.
// contrib[kk] is group kk's contribution (one source per group on the NCCL paths); own_k's may be fp32.
void adam_update(const Unit& u, const void* const* contrib, int n_contrib, int own_k, bool own_f32) {
  GradSources src;
  src.n_groups = n_contrib;
  for (int kk = 0; kk < n_contrib; ++kk) {
    src.p[kk] = contrib[kk];
    src.group_end[kk] = kk + 1;
    if (kk == own_k && own_f32) src.f32_mask |= 1u << kk;
  }
  adam_apply(u, src, n_contrib);
}

AdamParams adam_params() {
  AdamParams hp;
  hp.lr = g->dims.lr;
  hp.beta1 = g->dims.beta1;
  hp.beta2 = g->dims.beta2;
  hp.eps = g->dims.adam_eps;
  hp.wd = g->dims.weight_decay;
  hp.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(g->dims.beta1), g->step_t));
  hp.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(g->dims.beta2), g->step_t));
  return hp;
}

void adam_apply(const Unit& u, const GradSources& src, int n_src) {
  cudaStream_t s = g->gs;
  AdamRanges nd;
  for (int r = 0; r < u.n_nd; ++r) {
    nd.lo[r] = u.nd_lo[r];
    nd.hi[r] = u.nd_hi[r];
  }
  // algorithmic bytes: the sources (fp32 4 B or wire) + master/m/v read 12 B + master/m/v/wire written 12 B + esz
  double src_bytes = 0;
  for (int si = 0; si < n_src; ++si) src_bytes += (src.f32_mask >> si & 1u) ? 4.0 : static_cast<double>(g->esz);
  Timed t(s, 2, (src_bytes + 24.0 + g->esz) * u.s);
  BY_TYPE(adamw_grouped<float>(src, g->master + u.off, g->mom + u.off, g->vel + u.off, (float*)wptr(g->wire, u.off),
                               u.s, u.lo, nd, adam_params(), s),
          adamw_grouped<bf16>(src, g->master + u.off, g->mom + u.off, g->vel + u.off, (bf16*)wptr(g->wire, u.off),
                              u.s, u.lo, nd, adam_params(), s));
}

// ------------------------------------------------------------------------------------ NVLink peer path (GWPS)
// Replaces the NCCL collectives of the striped schedule when every rank could map every peer (peer.cu):
//   a3  rank (k, j) pulls stripe j of a remote unit from its owner (k_o, j)'s wire copy (the rail transfer), then
//       the other G−1 stripes from its group members (from their wire copies when the group owns the unit, else
//       from the slot each member filled over its own rail) -- plain cudaMemcpyAsync calls, run by copy engines;
//   a8  the members' fp32 gradient accumulators are read in place over NVLink: a non-owner group's member j sums
//       stripe j over its group into a wire-dtype rail partial; the owner's member j reads its group's G fp32
//       stripes and the D−1 rail partials inside
//   a9  the fused accumulate + AdamW kernel.
// Every cross-rank dependency is a sequence flag (RAW: "ready", WAR: "done reading"); the step-end loss all-reduce
// orders one step's owner updates before the next step's pulls.
inline int rank_of(int k, int j) { return k * g->G + j; }
bool fault_gdone_plus1() {
  static const bool on = [] {
    const char* e = std::getenv("TAWPIPE_FAULT");
    return e && std::string(e) == "gdone+1";
  }();
  return on;
}
// test-only fault (TAWPIPE_FAULT=skip-e-gather): the peer path's E gather leaves the ledger unaccounted, as a schedule
// that dropped that transfer would -- the end-of-step ledger = plan check must fail the step
bool fault_skip_e_gather() {
  static const bool on = [] {
    const char* e = std::getenv("TAWPIPE_FAULT");
    return e && std::string(e) == "skip-e-gather";
  }();
  return on;
}
inline uint32_t* flag_at(int dst_rank, int kind, int src_rank) {
  return static_cast<uint32_t*>(g->peer[dst_rank][PB_SIG]) + kind * kSigRanks + src_rank;
}
inline const uint32_t* my_flag(int kind, int src_rank) { return g->sig + kind * kSigRanks + src_rank; }
inline char* peer_ptr(int rank, int buf, int64_t bytes) { return static_cast<char*>(g->peer[rank][buf]) + bytes; }

// tell every other member of my group: flag `kind` from me is now `seq`
// Group members run the same gather / reduction sequence over the same ownership, so what I send a member of a
// group-level kind is exactly what it sends me: record it as the value my flag from that member must end at.
void expect_flag(int kind, int src, uint32_t seq) {
  uint32_t& e = g->sig_expect[static_cast<size_t>(kind) * kSigRanks + src];
  e = std::max(e, seq);
}
void signal_group(int kind, uint32_t seq, cudaStream_t s) {
  uint32_t* f[kMaxSignalTargets];
  int n = 0;
  for (int jj = 0; jj < g->G; ++jj)
    if (jj != g->j) {
      f[n++] = flag_at(rank_of(g->k, jj), kind, g->rank);
      expect_flag(kind, rank_of(g->k, jj), seq);
    }
  signal_peers(f, n, seq, s);
}
void wait_group_peers(int kind, uint32_t seq, cudaStream_t s) {
  if (g->G == 1) return;
  if (s == g->cs && g->timing) {   // a compute-stream wait on peers is exposed communication
    Timed t(s, 3, 0);
    for (int jj = 0; jj < g->G; ++jj)
      if (jj != g->j) wait_flag(my_flag(kind, rank_of(g->k, jj)), seq, s);
    return;
  }
  for (int jj = 0; jj < g->G; ++jj)
    if (jj != g->j) wait_flag(my_flag(kind, rank_of(g->k, jj)), seq, s);
}

int weight_pbuf(const Unit& u, int slot) {
  return u.cls == U_E ? PB_EBUF : u.cls == U_F ? PB_FBUF : (slot ? PB_WBUF1 : PB_WBUF0);
}

void copy_stripe(void* dst, const void* src, int64_t bytes, cudaStream_t s) {
  Timed t(s, 5, static_cast<double>(bytes));
  TP_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, s));
}

void gather_p2p(int uid, int slot) {
  Ctx& c = *g;
  const Unit& u = c.units[uid];
  cudaStream_t s = c.ws;
  const uint32_t seq = ++c.wseq;
  const int64_t sb = u.s * static_cast<int64_t>(c.esz);   // stripe bytes
  char* dst = static_cast<char*>(unit_buffer(uid, slot));
  const int pb = weight_pbuf(u, slot);
  if (u.cls == U_BLOCK) {
    // WAR: if the members pulled the previous layer of this slot from my rail stripe, they must be done with it
    if (c.wprev[slot]) wait_group_peers(SK_WDONE, c.wprev[slot], s);
    c.wprev[slot] = (!u.owned && c.G > 1) ? seq : 0;
  }
  if (!u.owned) {   // rail: stripe j from the owner group's member j
    const int src = rank_of(u.owner, c.j);
    copy_stripe(dst + c.j * sb, peer_ptr(src, PB_WIRE, c.gofs[static_cast<size_t>(u.owner) * (c.L + 2) + uid] * c.esz),
                sb, s);
    if (emu_rail_crosses()) {
      Timed t(s, 5, 0);
      emu_delay(static_cast<double>(c.D - 1) * u.s * c.esz, s);
    }
    if (c.G > 1) signal_group(SK_RAIL, seq, s);
  } else {
    if (c.G > 1) copy_stripe(dst + c.j * sb, wptr(c.wire, u.off), sb, s);   // my own stripe into the layer buffer
    if (emu_rail_crosses()) {   // emulated link: the owner's link carries its stripe to the D − 1 other groups
      Timed t(s, 5, 0);
      emu_delay(static_cast<double>(c.D - 1) * u.s * c.esz, s);
    }
  }
  for (int jj = 0; jj < c.G; ++jj) {   // intra-group: the other stripes from the members
    if (jj == c.j) continue;
    const int src = rank_of(c.k, jj);
    if (u.owned) {
      copy_stripe(dst + jj * sb, peer_ptr(src, PB_WIRE, u.off * static_cast<int64_t>(c.esz)), sb, s);
    } else {
      wait_flag(my_flag(SK_RAIL, src), seq, s);
      copy_stripe(dst + jj * sb, peer_ptr(src, pb, jj * sb), sb, s);
    }
  }
  if (c.G > 1 && emu_group_crosses()) {
    Timed t(s, 5, 0);
    emu_delay(static_cast<double>(c.G - 1) * u.s * c.esz, s);
  }
  if (c.G > 1 && !u.owned && u.cls == U_BLOCK) signal_group(SK_WDONE, seq, s);
  c.nvl_w_bytes += static_cast<double>(u.owned ? c.G - 1 : c.G) * sb;
  if (!(u.cls == U_E && fault_skip_e_gather())) ledger_gather(u, c.G, c.D, c.ledger);
}

void reduce_p2p(int uid, int slot, float* gacc) {
  Ctx& c = *g;
  const Unit& u = c.units[uid];
  cudaStream_t s = c.gs;
  const uint32_t seq = ++c.gseq;
  const int gb = u.cls == U_E ? PB_GACCE : u.cls == U_F ? PB_GACCF : (slot ? PB_GACC1 : PB_GACC0);
  const int ps = u.cls == U_E ? 2 : u.cls == U_F ? 3 : slot;          // rail partial slot
  const int64_t stripe_b = static_cast<int64_t>(c.j) * u.s * 4;      // my stripe inside an fp32 accumulator
  const int64_t part_b = static_cast<int64_t>(ps) * c.max_s * c.esz;
  if (u.cls == U_BLOCK) c.gprev[slot] = seq;
  if (c.G > 1) {
    signal_group(SK_GREADY, seq, s);   // my accumulator for this unit is complete
    wait_group_peers(SK_GREADY, seq, s);
  }
  if (u.owned) {
    // emulated link (NEXT-3): the owner's rail link receives the D − 1 partials while their senders transmit, so
    // its delay runs before it waits for them (in parallel with theirs, as the NCCL path's send / recv pair did)
    if (emu_rail_crosses()) {
      Timed t(s, 6, 0);
      emu_delay(static_cast<double>(c.D - 1) * u.s * c.esz, s);
    }
    if (emu_group_crosses()) {
      Timed t(s, 6, 0);
      emu_delay(static_cast<double>(c.G - 1) * u.s * 4, s);
    }
    GradSources src;
    int n = 0;
    for (int kk = 0; kk < c.D; ++kk) {   // ascending group order (R16)
      if (kk == c.k) {
        for (int jj = 0; jj < c.G; ++jj) {   // member order
          src.p[n] = peer_ptr(rank_of(c.k, jj), gb, stripe_b);
          src.f32_mask |= 1u << n;
          ++n;
        }
      } else {
        wait_flag(my_flag(SK_PREADY, rank_of(kk, c.j)), seq, s);
        expect_flag(SK_PREADY, rank_of(kk, c.j), seq);
        src.p[n++] = peer_ptr(rank_of(kk, c.j), PB_PART, part_b);
      }
      src.group_end[src.n_groups++] = n;
    }
    adam_apply(u, src, n);
    c.nvl_g_bytes += (4.0 * (c.G - 1) + static_cast<double>(c.esz) * (c.D - 1)) * u.s;
    if (c.G > 1 && u.cls == U_E && c.j == 0 && fault_gdone_plus1()) {
      // test-only fault (TAWPIPE_FAULT=gdone+1): member 0 mis-numbers its last GDONE of the step by one; waits are
      // "≥", so nothing blocks -- exactly the silent class of protocol error the end-of-step check must catch
      uint32_t* f[kMaxSignalTargets];
      int nf = 0;
      for (int jj = 1; jj < c.G; ++jj) {
        f[nf++] = flag_at(rank_of(c.k, jj), SK_GDONE, c.rank);
        expect_flag(SK_GDONE, rank_of(c.k, jj), seq);
      }
      signal_peers(f, nf, seq + 1, s);
    } else if (c.G > 1) {
      signal_group(SK_GDONE, seq, s);
    }
    uint32_t* f[kMaxSignalTargets];
    int nf = 0;
    for (int kk = 0; kk < c.D; ++kk)
      if (kk != c.k) f[nf++] = flag_at(rank_of(kk, c.j), SK_PDONE, c.rank);
    signal_peers(f, nf, seq, s);
  } else {
    const int owner = rank_of(u.owner, c.j);
    // WAR: the owner that read the previous partial in this slot (layers alternate owners) is done with it
    if (c.pprev[ps]) wait_flag(my_flag(SK_PDONE, c.pprev_owner[ps]), c.pprev[ps], s);
    c.pprev[ps] = seq;
    c.pprev_owner[ps] = owner;
    expect_flag(SK_PDONE, owner, seq);   // the owner acknowledges every partial it reads
    PartialSources src;
    for (int jj = 0; jj < c.G; ++jj) src.p[src.n++] = reinterpret_cast<const float*>(peer_ptr(rank_of(c.k, jj), gb, stripe_b));
    {
      Timed t(s, 6, (4.0 * c.G + c.esz) * u.s);
      BY_TYPE(group_partial<float>(src, reinterpret_cast<float*>(static_cast<char*>(c.part) + part_b), u.s, s),
              group_partial<bf16>(src, reinterpret_cast<bf16*>(static_cast<char*>(c.part) + part_b), u.s, s));
      if (emu_group_crosses()) emu_delay(static_cast<double>(c.G - 1) * u.s * 4, s);
      // emulated link: the rail exchange that delivers this partial to the owner (as on the NCCL path)
      if (emu_rail_crosses()) emu_delay(static_cast<double>(c.D - 1) * u.s * c.esz, s);
    }
    c.nvl_g_bytes += 4.0 * (c.G - 1) * u.s;
    uint32_t* f = flag_at(owner, SK_PREADY, c.rank);
    signal_peers(&f, 1, seq, s);
    if (c.G > 1) signal_group(SK_GDONE, seq, s);
  }
  ledger_reduce(u, c.G, c.D, c.ledger);
}

void wait_on(cudaStream_t s, cudaEvent_t e) {
  if (s == g->cs && g->timing) {
    Timed t(s, 3, 0);
    TP_CUDA(cudaStreamWaitEvent(s, e, 0));
  } else {
    TP_CUDA(cudaStreamWaitEvent(s, e, 0));
  }
}

// ------------------------------------------------------------------------------------ layer compute (a5, a7)
struct LayerW {
  const void *attn_norm, *wqkv, *wo, *mlp_norm, *wgu, *wdown;
};
LayerW layer_weights(void* W) {
  const int64_t H = g->H, I = g->I;
  LayerW w;
  w.attn_norm = wptr(W, 0);
  w.wqkv = wptr(W, H);
  w.wo = wptr(W, H + 3 * H * H);
  w.mlp_norm = wptr(W, H + 4 * H * H);
  w.wgu = wptr(W, 2 * H + 4 * H * H);
  w.wdown = wptr(W, 2 * H + 4 * H * H + 2 * I * H);
  return w;
}

Acts& acts_for(int l, int mb) { return g->dims.ckpt ? g->acts[0] : g->acts[static_cast<size_t>(l) * g->m + mb]; }
// the activations of (l, mb) as the layer's forward / backward see them: kept tensors where selective
// checkpointing kept them, else the scratch set (ckpt) or the per-layer set (no ckpt)
struct View {
  void *a, *qkv, *o, *h1, *b, *gu, *y;
  float *r1, *lse, *r2;
  uint8_t keep;
};
View view(int l, int mb) {
  const Acts& A = acts_for(l, mb);
  View v{A.a, A.qkv, A.o, A.h1, A.b, A.gu, A.y, A.r1, A.lse, A.r2, 0};
  if (!g->kept.empty()) {
    const Kept& k = g->kept[static_cast<size_t>(l) * g->m + mb];
    v.keep = k.flags;
    if (k.flags & KEEP_ATTN) {
      v.o = k.o;
      v.lse = k.lse;
    }
    if (k.flags & KEEP_QKV) v.qkv = k.qkv;
    if (k.flags & KEEP_H1) v.h1 = k.h1;
    if (k.flags & KEEP_MLP) v.gu = k.gu;   // y stays in the scratch set (re-derived from gu in the recompute)
  }
  return v;
}
void* ck(int l, int mb) { return g->ck[static_cast<size_t>(l) * g->m + mb]; }

void layer_forward(int l, int mb, void* W, bool write_out) {
  cudaStream_t s = g->cs;
  const int64_t T = g->T, H = g->H, I = g->I;
  LayerW w = layer_weights(W);
  const View A = view(l, mb);
  void* hin = ck(l, mb);
  // the recompute pass (write_out false) skips every step whose output selective checkpointing kept
  const uint8_t skip = write_out ? 0 : A.keep;
  double work = 0;
  k_rmsnorm_fwd(hin, w.attn_norm, A.a, A.r1, T, s);
  if (!(skip & KEEP_QKV)) {
    if (g->rope_cs != nullptr) {   // bf16 tcgen05 path: RoPE of q | k applied in the GEMM's epilogue
      GemmArgs a{T, 3 * H, H, A.a, H, true, w.wqkv, H, true, A.qkv, 3 * H, false, false, nullptr};
      a.rope.cs = g->rope_cs;
      a.rope.S = g->S;
      a.rope.dh = g->dh;
      a.rope.cols = 2 * H;
      Timed t(s, 0, 2.0 * T * 3 * H * H);
      gemm_tc_bf16(a, s);
    } else {
      gemm(T, 3 * H, H, A.a, H, true, w.wqkv, H, true, A.qkv, 3 * H, false, false, nullptr, s);
      k_rope(A.qkv, false, s);
    }
    work += 2.0 * T * 3 * H * H;
  }
  if (!(skip & KEEP_ATTN)) {
    attn_fwd(A.qkv, A.o, A.lse, s);
    work += attn_flops_fwd();
  }
  if (!(skip & KEEP_H1)) {
    gemm(T, H, H, A.o, H, true, w.wo, H, true, A.h1, H, false, false, hin, s);
    work += 2.0 * T * H * H;
  }
  k_rmsnorm_fwd(A.h1, w.mlp_norm, A.b, A.r2, T, s);
  if (!(skip & KEEP_MLP)) {
    work += 2.0 * T * 2 * I * H;
    if (g->bf && !gemm_force_simt()) {
      // gate/up GEMM with the SwiGLU epilogue: y directly; gu is stored only when a backward will read it
      // (no checkpointing, the recompute pass, a kept MLP, or the last layer's last micro-batch which skips
      // recompute)
      const bool need_gu = !g->dims.ckpt || !write_out || (A.keep & KEEP_MLP) || (l == g->L - 1 && mb == g->m - 1);
      GemmArgs a{T, 2 * I, H, A.b, H, true, w.wgu, H, true, need_gu ? A.gu : nullptr, 2 * I, false, false, nullptr};
      a.epi = 3;
      a.aux = A.y;
      a.ldx = I;
      a.I = I;
      Timed t(s, 0, 2.0 * T * 2 * I * H);
      gemm_tc_bf16(a, s);
    } else {
      gemm(T, 2 * I, H, A.b, H, true, w.wgu, H, true, A.gu, 2 * I, false, false, nullptr, s);
      Timed t(s, 4, 0);
      BY_TYPE(swiglu_fwd<float>((const float*)A.gu, (float*)A.y, T, (int)I, s),
              swiglu_fwd<bf16>((const bf16*)A.gu, (bf16*)A.y, T, (int)I, s));
    }
  } else {   // recompute with a kept gu: y = SwiGLU(gu) for the down projection's wgrad
    Timed t(s, 4, 0);
    BY_TYPE(swiglu_fwd<float>((const float*)A.gu, (float*)A.y, T, (int)I, s),
            swiglu_fwd<bf16>((const bf16*)A.gu, (bf16*)A.y, T, (int)I, s));
  }
  if (write_out) gemm(T, H, I, A.y, I, true, w.wdown, I, true, ck(l + 1, mb), H, false, false, A.h1, s);
  if (!write_out) g->recompute_gflop += work * 1e-9;
}

// Gradient accumulators are not zeroed by a full memset per layer: the first micro-batch's wgrad GEMMs store
// (EPI_F32_STORE) and the later ones accumulate; only the two RMSNorm-gain ranges (which the norm backward adds
// into) are zeroed (gacc_store_first).  0 + x == x in fp32, so the values are identical to memset + accumulate.
bool gacc_store_first() {
  static const bool on = [] {
    const char* e = std::getenv("TAWPIPE_GACC_ZERO");
    return !(e && std::string(e) == "memset");
  }();
  return on;
}

void layer_backward(int l, int mb, void* W, float* G_, bool first) {
  cudaStream_t s = g->cs;
  const bool acc = !(first && gacc_store_first());
  const int64_t T = g->T, H = g->H, I = g->I;
  LayerW w = layer_weights(W);
  // recompute from the checkpoint h_l; the last layer's last micro-batch is still resident in the
  // scratch activations from the forward pass, so it needs no recompute
  if (g->dims.ckpt && !(l == g->L - 1 && mb == g->m - 1)) layer_forward(l, mb, W, false);
  const View A = view(l, mb);
  void* hin = ck(l, mb);
  void* dh = g->dhb[mb];
  float* gq = G_ + H;                      // Wq|Wk|Wv  [3H, H]
  float* go = G_ + H + 3 * H * H;          // Wo        [H, H]
  float* gmn = G_ + H + 4 * H * H;         // mlp_norm  [H]
  float* ggu = G_ + 2 * H + 4 * H * H;     // Wgate|Wup [2I, H]
  float* gd = G_ + 2 * H + 4 * H * H + 2 * I * H;  // Wdown [H, I]
  // h2 = h1 + y·Wdownᵀ
  gemm(H, I, T, dh, H, false, A.y, I, false, gd, I, true, acc, nullptr, s);
  if (g->bf && !gemm_force_simt()) {
    // dgrad of the down projection with the SwiGLU backward in the epilogue: dY never reaches HBM
    GemmArgs a{T, I, H, dh, H, true, w.wdown, I, false, g->dGU, 2 * I, false, false, nullptr};
    a.epi = 4;
    a.aux = A.gu;
    a.ldx = 2 * I;
    a.I = I;
    Timed t(s, 0, 2.0 * T * I * H);
    gemm_tc_bf16(a, s);
  } else {
    gemm(T, I, H, dh, H, true, w.wdown, I, false, g->dY, I, false, false, nullptr, s);
    Timed t(s, 4, 0);
    BY_TYPE(swiglu_bwd<float>((const float*)g->dY, (const float*)A.gu, (float*)g->dGU, T, (int)I, s),
            swiglu_bwd<bf16>((const bf16*)g->dY, (const bf16*)A.gu, (bf16*)g->dGU, T, (int)I, s));
  }
  gemm(2 * I, H, T, g->dGU, 2 * I, false, A.b, H, false, ggu, H, true, acc, nullptr, s);
  gemm(T, H, 2 * I, g->dGU, 2 * I, true, w.wgu, H, false, g->db, H, false, false, nullptr, s);
  k_rmsnorm_bwd(g->db, A.h1, w.mlp_norm, A.r2, dh, g->dh1, gmn, T, s);
  // h1 = h + o·Woᵀ
  gemm(H, H, T, g->dh1, H, false, A.o, H, false, go, H, true, acc, nullptr, s);
  gemm(T, H, H, g->dh1, H, true, w.wo, H, false, g->dO, H, false, false, nullptr, s);
  attn_bwd(A.qkv, A.o, A.lse, g->dO, g->dqkv, s);
  if (!use_tc_attention()) k_rope(g->dqkv, true, s);   // the tcgen05 backward applies it in its epilogues
  gemm(3 * H, H, T, g->dqkv, 3 * H, false, A.a, H, false, gq, H, true, acc, nullptr, s);
  gemm(T, H, 3 * H, g->dqkv, 3 * H, true, w.wqkv, H, false, g->da, H, false, false, nullptr, s);
  k_rmsnorm_bwd(g->da, hin, w.attn_norm, A.r1, g->dh1, dh, G_, T, s);
}

// a6: final RMSNorm + LM head + cross-entropy, forward and backward back to back, in row chunks
void head(int mb, void* F, float* GF) {
  cudaStream_t s = g->cs;
  const int64_t T = g->T, H = g->H, V = g->V;
  const void* gf = F;
  const void* Wh = wptr(F, H);
  void* hL = ck(g->L, mb);
  k_rmsnorm_fwd(hL, gf, g->fnorm, g->rstd_f, T, s);
  const float inv_denom = 1.0f / static_cast<float>(static_cast<double>(g->N) * g->Bm * g->S);
  for (int64_t c0 = 0; c0 < T; c0 += g->Tc) {
    const int64_t tc = (T - c0) < g->Tc ? (T - c0) : g->Tc;
    void* fc = wptr(g->fnorm, c0 * H);
    gemm(tc, V, H, fc, H, true, Wh, H, true, g->logits, V, false, false, nullptr, s);
    {
      Timed t(s, 4, 0);
      const int32_t* tg = g->d_tgt + static_cast<int64_t>(mb) * T + c0;
      BY_TYPE(cross_entropy<float>((float*)g->logits, tg, tc, (int)V, inv_denom, g->loss_rows + c0, s),
              cross_entropy<bf16>((bf16*)g->logits, tg, tc, (int)V, inv_denom, g->loss_rows + c0, s));
    }
    const bool acc = !(mb == 0 && c0 == 0 && gacc_store_first());   // the first chunk stores (see layer_backward)
    gemm(V, H, tc, g->logits, V, false, fc, H, false, GF + H, H, true, acc, nullptr, s);
    gemm(tc, H, V, g->logits, V, true, Wh, H, false, wptr(g->df, c0 * H), H, false, false, nullptr, s);
  }
  k_rmsnorm_bwd(g->df, hL, gf, g->rstd_f, nullptr, g->dhb[mb], GF, T, s);
  sum_f32_to_f64(g->loss_rows, T, g->d_loss, s);
}

__global__ void split_tokens_kernel(const int32_t* __restrict__ tok, int64_t seqs, int S, int32_t* __restrict__ in,
                                    int32_t* __restrict__ tgt) {
  const int64_t n = seqs * S;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = i / S, p = i % S;
    in[i] = tok[q * (S + 1) + p];
    tgt[i] = tok[q * (S + 1) + p + 1];
  }
}

// ------------------------------------------------------------------------------------ trace export (NEXT-4)
// Trace-Event JSON ("X" complete events, microseconds from the step's first compute-stream event) of the last
// timed step: one thread per stream (0 compute, 1 weights, 2 gradients), pid = rank.  otherData carries the
// step time and, per stream, the busy time (union of its regions) and the compute stream's idle ("bubble")
// fraction: time the compute stream is neither running a timed kernel nor waiting on communication.
void build_trace_json(float step_ms) {
  Ctx& c = *g;
  static const char* kind_name[7] = {"gemm", "attention", "adamw", "exposed_comm_wait", "elementwise",
                                     "weight_comm", "grad_comm"};
  std::vector<std::array<double, 2>> iv[3];
  std::string out;
  out.reserve(c.regions.size() * 128 + 512);
  out += "{\"traceEvents\":[";
  char buf[256];
  bool first = true;
  for (auto& r : c.regions) {
    float t0 = 0.f, t1 = 0.f;
    TP_CUDA(cudaEventElapsedTime(&t0, c.ev_s0, r.a));
    TP_CUDA(cudaEventElapsedTime(&t1, c.ev_s0, r.b));
    if (r.kind != 3) iv[r.stream].push_back({static_cast<double>(t0), static_cast<double>(t1)});
    std::snprintf(buf, sizeof(buf),
                  "%s{\"name\":\"%s\",\"cat\":\"tawpipe\",\"ph\":\"X\",\"ts\":%.3f,\"dur\":%.3f,\"pid\":%d,"
                  "\"tid\":%d,\"args\":{\"work\":%.6g}}",
                  first ? "" : ",", kind_name[r.kind], t0 * 1e3, (t1 - t0) * 1e3, c.rank, r.stream, r.work);
    out += buf;
    first = false;
  }
  double busy[3] = {0, 0, 0};
  for (int st = 0; st < 3; ++st) {  // union of intervals
    auto& v = iv[st];
    std::sort(v.begin(), v.end());
    double cur0 = -1, cur1 = -1;
    for (auto& x : v) {
      if (x[0] > cur1) {
        if (cur1 > cur0) busy[st] += cur1 - cur0;
        cur0 = x[0];
        cur1 = x[1];
      } else if (x[1] > cur1) {
        cur1 = x[1];
      }
    }
    if (cur1 > cur0) busy[st] += cur1 - cur0;
  }
  std::snprintf(buf, sizeof(buf),
                "],\"displayTimeUnit\":\"ms\",\"otherData\":{\"rank\":%d,\"step\":%d,\"step_ms\":%.4f,"
                "\"busy_ms\":[%.4f,%.4f,%.4f],\"exposed_comm_ms\":%.4f,\"compute_idle_frac\":%.6f}}",
                c.rank, c.step_t, step_ms, busy[0], busy[1], busy[2], c.stats[1],
                step_ms > 0 ? std::max(0.0, 1.0 - (busy[0] + c.stats[1]) / step_ms) : 0.0);
  out += buf;
  c.trace_json.swap(out);
}

// Invariant of the peer path, checked after every step (the step ends with a device-wide barrier, so no flag can
// still be in flight): every flag a peer writes into this rank ends at exactly the last sequence number of its
// kind that peer had to send.  A lost, duplicated or mis-numbered signal -- a protocol race -- raises
// TAWPIPE_EINVARIANT instead of silently mis-ordering a later step.
void check_flags() {
  Ctx& c = *g;
  std::vector<uint32_t> host(static_cast<size_t>(SK_N) * kSigRanks);
  TP_CUDA(cudaMemcpy(host.data(), c.sig, host.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  static const char* names[SK_N] = {"RAIL", "WDONE", "GREADY", "GDONE", "PREADY", "PDONE"};
  for (int kind = 0; kind < SK_N; ++kind)
    for (int src = 0; src < c.P; ++src) {
      const size_t i = static_cast<size_t>(kind) * kSigRanks + src;
      if (c.sig_expect[i] != 0 && host[i] != c.sig_expect[i])
        throw Error(TAWPIPE_EINVARIANT, std::string("peer flag ") + names[kind] + " from rank " + std::to_string(src) +
                                            " is " + std::to_string(host[i]) + ", expected " +
                                            std::to_string(c.sig_expect[i]) + " at the end of step " +
                                            std::to_string(c.step_t));
    }
}

// ------------------------------------------------------------------------------------ one iteration
double run_step(const int32_t* tokens, bool device_tokens) {
  Ctx& c = *g;
  c.step_t += 1;
  std::memset(c.ledger, 0, sizeof(c.ledger));
  c.regions.clear();
  c.recompute_gflop = 0;
  c.nvl_w_bytes = c.nvl_g_bytes = 0;
  c.ev_used = 0;
  c.launches_at_start = g_kstats.launches;
  const int64_t seqs = static_cast<int64_t>(c.m) * c.Bm;
  const int64_t tok_elems = seqs * (c.S + 1);
  TRACE("step %d begin (device tokens %d)\n", c.step_t, device_tokens ? 1 : 0);
  TP_CUDA(cudaEventRecord(c.ev_s0, c.cs));
  TP_CUDA(cudaEventRecord(c.ev_ws0, c.ws));
  TP_CUDA(cudaEventRecord(c.ev_gs0, c.gs));
  if (device_tokens) {
    TP_CUDA(cudaMemcpyAsync(c.d_tok, tokens, tok_elems * 4, cudaMemcpyDeviceToDevice, c.cs));
  } else {
    const int32_t* mine = tokens + static_cast<int64_t>(c.rank) * tok_elems;  // contiguous m micro-batches (R4)
    std::memcpy(c.h_tok, mine, tok_elems * 4);
    TP_CUDA(cudaMemcpyAsync(c.d_tok, c.h_tok, tok_elems * 4, cudaMemcpyHostToDevice, c.cs));
  }
  split_tokens_kernel<<<256, 256, 0, c.cs>>>(c.d_tok, seqs, c.S, c.d_in, c.d_tgt);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
  TP_CUDA(cudaMemsetAsync(c.d_loss, 0, sizeof(double), c.cs));
  if (trace_on()) {
    TP_CUDA(cudaDeviceSynchronize());
    TRACE("tokens staged\n");
  }
  const bool cco = !(c.dims.schedule & TAWPIPE_NO_CCO);
  const int E = c.L, F = c.L + 1;
  // ws / gs start after cs has seen the tokens (keeps all three streams inside the timed step)
  TP_CUDA(cudaEventRecord(c.evGE, c.cs));
  TP_CUDA(cudaStreamWaitEvent(c.ws, c.evGE, 0));
  TP_CUDA(cudaStreamWaitEvent(c.gs, c.evGE, 0));

  // ---- E: gather (forward only), embed (a4)
  void* Ebuf = unit_buffer(E, 0);
  gather(E, 0);
  TP_CUDA(cudaEventRecord(c.evE, c.ws));
  wait_on(c.cs, c.evE);
  for (int mb = 0; mb < c.m; ++mb) {
    Timed t(c.cs, 4, 0);
    BY_TYPE(embed_fwd<float>(c.d_in + static_cast<int64_t>(mb) * c.T, c.S, c.Bm, c.S, (const float*)Ebuf, c.H,
                             (float*)ck(0, mb), c.cs),
            embed_fwd<bf16>(c.d_in + static_cast<int64_t>(mb) * c.T, c.S, c.Bm, c.S, (const bf16*)Ebuf, c.H,
                            (bf16*)ck(0, mb), c.cs));
  }
  // ---- forward with CCO prefetch (a3, a5)
  gather(0, 0);
  TP_CUDA(cudaEventRecord(c.w_ready[0], c.ws));
  for (int l = 0; l < c.L; ++l) {
    const int slot = l & 1;
    if (cco && l + 1 < c.L) {
      TP_CUDA(cudaStreamWaitEvent(c.ws, c.w_free[(l + 1) & 1], 0));
      gather(l + 1, (l + 1) & 1);
      TP_CUDA(cudaEventRecord(c.w_ready[(l + 1) & 1], c.ws));
    }
    if (l == c.L - 1) {  // F lives in its own buffer: prefetch it during the last layer
      gather(F, 0);
      TP_CUDA(cudaEventRecord(c.evF, c.ws));
    }
    wait_on(c.cs, c.w_ready[slot]);
    check_slot(l, slot);
    void* W = unit_buffer(l, slot);
    TRACE("forward layer %d\n", l);
    for (int mb = 0; mb < c.m; ++mb) layer_forward(l, mb, W, true);
    TP_CUDA(cudaEventRecord(c.w_free[slot], c.cs));
    if (!cco && l + 1 < c.L) {  // ablation: transfer serialised after the compute of the current step
      TP_CUDA(cudaStreamWaitEvent(c.ws, c.w_free[slot], 0));
      gather(l + 1, (l + 1) & 1);
      TP_CUDA(cudaEventRecord(c.w_ready[(l + 1) & 1], c.ws));
    }
  }
  // ---- head F (a6)
  wait_on(c.cs, c.evF);
  if (gacc_store_first())
    TP_CUDA(cudaMemsetAsync(c.gaccF, 0, c.H * 4, c.cs));   // final-norm gain (the norm backward adds into it)
  else
    TP_CUDA(cudaMemsetAsync(c.gaccF, 0, c.units[F].n_pad * 4, c.cs));
  void* Fbuf = unit_buffer(F, 0);
  for (int mb = 0; mb < c.m; ++mb) head(mb, Fbuf, c.gaccF);
  TP_CUDA(cudaEventRecord(c.evGF, c.cs));
  wait_on(c.gs, c.evGF);
  reduce_and_update(F, 0, c.gaccF);
  // ---- backward (a7) with prefetch of l-1, gradient reduction + AdamW on gs (a8, a9)
  for (int l = c.L - 1; l >= 0; --l) {
    const int slot = l & 1;
    if (cco && l - 1 >= 0) {
      TP_CUDA(cudaStreamWaitEvent(c.ws, c.w_free[(l - 1) & 1], 0));
      gather(l - 1, (l - 1) & 1);
      TP_CUDA(cudaEventRecord(c.w_ready[(l - 1) & 1], c.ws));
    }
    if (l != c.L - 1) wait_on(c.cs, c.w_ready[slot]);  // r = 1: layer L-1 reuses its forward buffer (R12)
    wait_on(c.cs, c.g_free[slot]);
    if (c.p2p && c.gprev[slot]) wait_group_peers(SK_GDONE, c.gprev[slot], c.cs);   // peers done reading it
    if (gacc_store_first()) {   // the two norm gains; the weight matrices are stored by the first micro-batch
      TP_CUDA(cudaMemsetAsync(c.gacc[slot], 0, c.H * 4, c.cs));
      TP_CUDA(cudaMemsetAsync(c.gacc[slot] + c.H + 4 * static_cast<int64_t>(c.H) * c.H, 0, c.H * 4, c.cs));
    } else {
      TP_CUDA(cudaMemsetAsync(c.gacc[slot], 0, c.units[l].n_pad * 4, c.cs));
    }
    check_slot(l, slot);
    void* W = unit_buffer(l, slot);
    TRACE("backward layer %d\n", l);
    for (int mb = c.m - 1; mb >= 0; --mb) layer_backward(l, mb, W, c.gacc[slot], mb == c.m - 1);  // last first
    TP_CUDA(cudaEventRecord(c.w_free[slot], c.cs));
    TP_CUDA(cudaEventRecord(c.g_ready[slot], c.cs));
    if (!cco && l - 1 >= 0) {
      TP_CUDA(cudaStreamWaitEvent(c.ws, c.w_free[slot], 0));
      gather(l - 1, (l - 1) & 1);
      TP_CUDA(cudaEventRecord(c.w_ready[(l - 1) & 1], c.ws));
    }
    TP_CUDA(cudaStreamWaitEvent(c.gs, c.g_ready[slot], 0));
    reduce_and_update(l, slot, c.gacc[slot]);
    TP_CUDA(cudaEventRecord(c.g_free[slot], c.gs));
  }
  // ---- E backward: scatter-add into the fp32 accumulator, then reduce + update (a4, a8, a9)
  TP_CUDA(cudaMemsetAsync(c.gaccE, 0, c.units[E].n_pad * 4, c.cs));
  for (int mb = 0; mb < c.m; ++mb) {
    Timed t(c.cs, 4, 0);
    embed_bwd(c.d_in + static_cast<int64_t>(mb) * c.T, c.S, c.Bm, c.S, c.dhb[mb], !c.bf, c.H, c.V, c.gaccE,
              c.emb_scratch, c.emb_scratch_bytes, c.cs);
  }
  TP_CUDA(cudaEventRecord(c.evGE, c.cs));
  TP_CUDA(cudaStreamWaitEvent(c.gs, c.evGE, 0));
  reduce_and_update(E, 0, c.gaccE);
  // ---- a10: loss.  The all-reduce runs after this rank's weight and gradient streams joined the compute stream,
  // so its completion on any rank implies every rank finished every AdamW of the step: it is also the step
  // barrier that orders this step's owner updates before the next step's peer pulls of the wire copies.
  TP_CUDA(cudaEventRecord(c.ev_ws1, c.ws));
  TP_CUDA(cudaEventRecord(c.ev_gs1, c.gs));
  {
    // the compute stream's tail: waiting for the last reductions / AdamW and the loss all-reduce (which also waits for
    // the slowest rank) is exposed time of the step, accounted with the other exposed waits
    Timed t(c.cs, 3, 0);
    TP_CUDA(cudaStreamWaitEvent(c.cs, c.ev_ws1, 0));
    TP_CUDA(cudaStreamWaitEvent(c.cs, c.ev_gs1, 0));
    if (c.world > 1) TP_NCCL(ncclAllReduce(c.d_loss, c.d_loss, 1, ncclFloat64, ncclSum, c.world_comm, c.cs));
  }
  TP_CUDA(cudaMemcpyAsync(c.h_loss, c.d_loss, sizeof(double), cudaMemcpyDeviceToHost, c.cs));
  TP_CUDA(cudaEventRecord(c.ev_s1, c.cs));
  TP_CUDA(cudaStreamSynchronize(c.cs));
  TP_CUDA(cudaDeviceSynchronize());
  if (c.p2p) check_flags();
  for (int i = 0; i < TAWPIPE_LEDGER_N; ++i)   // the executed transfers are the planned schedule's, counter by counter
    TP_CHECK(c.ledger[i] == c.ledger_plan[i], TAWPIPE_EINVARIANT,
             "step ledger counter " + std::to_string(i) + " is " + std::to_string(c.ledger[i]) + ", the plan's " +
                 std::to_string(c.ledger_plan[i]));
  // ---- stats
  std::memset(c.stats, 0, sizeof(c.stats));
  float ms = 0.f;
  TP_CUDA(cudaEventElapsedTime(&ms, c.ev_s0, c.ev_s1));
  c.stats[0] = ms;
  if (c.timing) {
    for (auto& r : c.regions) {
      float e = 0.f;
      TP_CUDA(cudaEventElapsedTime(&e, r.a, r.b));
      switch (r.kind) {
        case 0: c.stats[4] += e; c.stats[5] += r.work * 1e-9; c.stats[6] += 1; break;
        case 1: c.stats[7] += e; c.stats[8] += r.work * 1e-9; break;
        case 2: c.stats[9] += e; c.stats[10] += r.work * 1e-9; break;
        case 3: c.stats[1] += e; break;
        case 4: c.stats[14] += e; break;
        case 5: c.stats[2] += e; break;
        case 6: c.stats[3] += e; break;
      }
    }
  }
  c.stats[11] = static_cast<double>(g_kstats.launches - c.launches_at_start);
  c.stats[12] = static_cast<double>(c.bytes_alloc) * 1e-9;
  c.stats[13] = static_cast<double>(c.esz);
  c.stats[15] = c.recompute_gflop;
  c.stats[16] = c.p2p ? 1.0 : 0.0;
  c.stats[17] = c.nvl_w_bytes * 1e-9;
  c.stats[18] = c.nvl_g_bytes * 1e-9;
  if (c.timing) build_trace_json(ms);
  return *c.h_loss / (static_cast<double>(c.N) * c.Bm * c.S);
}

// ------------------------------------------------------------------------------------ init
int64_t pad_to(int64_t n, int G) {
  const int64_t q = static_cast<int64_t>(G) * 64;
  return q * ((n + q - 1) / q);
}

void validate(int P, int G, int L, const tawpipe_dims* d, int N, int world) {
  TP_CHECK(d != nullptr, TAWPIPE_ECONFIG, "dims is NULL");
  TP_CHECK(P == world, TAWPIPE_ECONFIG, "n_devices (" + std::to_string(P) + ") != world size (" +
                                            std::to_string(world) + ")");
  TP_CHECK(G >= 1 && P % G == 0, TAWPIPE_ECONFIG, "P mod G != 0 (PAPER.md:53 requires P mod D = 0)");
  const int D = P / G;
  TP_CHECK(L >= 1 && L % D == 0, TAWPIPE_ECONFIG, "L mod D != 0 (striped DBS, reading R6)");
  TP_CHECK(N >= 1 && N % P == 0, TAWPIPE_ECONFIG, "N mod P != 0 (even micro-batch split, R4)");
  TP_CHECK(D <= 8, TAWPIPE_ECONFIG, "at most 8 groups");
  TP_CHECK(d->hidden > 0 && d->heads > 0 && d->hidden % d->heads == 0, TAWPIPE_ECONFIG, "H mod n_h != 0");
  TP_CHECK(d->ffn > 0 && d->vocab > 0 && d->seq > 0 && d->micro_bs > 0, TAWPIPE_ECONFIG, "non-positive dimension");
  TP_CHECK((d->hidden / d->heads) % 2 == 0, TAWPIPE_ECONFIG, "d_h must be even (rotate-half RoPE)");
  TP_CHECK(d->dtype == TAWPIPE_FP32 || d->dtype == TAWPIPE_BF16, TAWPIPE_ECONFIG, "dtype must be FP32 or BF16");
  TP_CHECK(d->reserved == 0, TAWPIPE_ECONFIG, "reserved must be 0");
  TP_CHECK(d->ckpt >= 0 && d->ckpt <= 2, TAWPIPE_ECONFIG, "ckpt must be 0, 1 or 2");
  TP_CHECK((d->schedule & ~(TAWPIPE_NO_CCO | TAWPIPE_RING | TAWPIPE_LITERAL)) == 0, TAWPIPE_ECONFIG,
           "unknown schedule flag");
  TP_CHECK(!((d->schedule & TAWPIPE_RING) && (d->schedule & TAWPIPE_LITERAL)), TAWPIPE_ECONFIG,
           "TAWPIPE_RING and TAWPIPE_LITERAL are exclusive");
  TP_CHECK(!(d->schedule & TAWPIPE_LITERAL) || L % P == 0, TAWPIPE_ECONFIG,
           "TAWPIPE_LITERAL needs L mod P == 0 (one whole shard per device, PAPER.md:123)");
  TP_CHECK(!(d->schedule & TAWPIPE_RING) || G == 1, TAWPIPE_ECONFIG,
           "TAWPIPE_RING owns whole layers per device: group_size must be 1");
  if (d->dtype == TAWPIPE_BF16) {
    const int dh = d->hidden / d->heads;
    TP_CHECK(dh == 64 || dh == 128, TAWPIPE_ECONFIG, "bf16 path: d_h must be 64 or 128");
    TP_CHECK(d->seq % 128 == 0, TAWPIPE_ECONFIG, "bf16 path: S mod 128 != 0");
    TP_CHECK(d->hidden % 128 == 0 && d->ffn % 128 == 0 && d->vocab % 128 == 0, TAWPIPE_ECONFIG,
             "bf16 path: H, I, V must be multiples of 128");
  }
}

// DBS plan (a1): units, ownership, stripes, canonical offsets, owned-state offsets of rank (k, j)
struct Plan {
  std::vector<Unit> units;
  int64_t owned_total = 0, max_pad = 0, max_s = 0;
};
// The per-step ledger of the documented schedule, written out as its own sequence (not by replaying run_step): E
// gather, forward gathers 0..L-1, F gather, F reduction, backward gathers L-2..0 (layer L-1 reuses its forward
// buffer, R12) with reductions L-1..0, E reduction.  tawpipe_plan returns it; every step checks its executed ledger
// against it (TAWPIPE_EINVARIANT), so a schedule change that skips or repeats a transfer fails loudly.
void plan_ledger(const Plan& pl, int P, int G, int L, int schedule, int rank, uint64_t* led) {
  const int D = P / G;
  const bool ring = (schedule & TAWPIPE_RING) != 0, literal = (schedule & TAWPIPE_LITERAL) != 0;
  auto gat = [&](const Unit& u) {
    if (ring) ledger_gather_ring(u, rank, P, led);
    else if (literal) ledger_gather_literal(u, G, D, rank / G, rank % G, led);
    else ledger_gather(u, G, D, led);
  };
  auto red = [&](const Unit& u) {
    if (ring) ledger_reduce_ring(u, rank, P, led);
    else if (literal) ledger_reduce_literal(u, G, D, rank / G, rank % G, led);
    else ledger_reduce(u, G, D, led);
  };
  gat(pl.units[L]);
  for (int l = 0; l < L; ++l) gat(pl.units[l]);
  gat(pl.units[L + 1]);
  red(pl.units[L + 1]);
  for (int l = L - 1; l >= 0; --l) {
    if (l != L - 1) gat(pl.units[l]);
    red(pl.units[l]);
  }
  red(pl.units[L]);
}

Plan make_plan(int P, int G, int L, int64_t H, int64_t I, int64_t V, int rank, bool literal) {
  Plan pl;
  const int D = P / G, k = rank / G, j = rank % G;
  const int64_t phi = 4 * H * H + 3 * H * I + 2 * H;
  pl.units.assign(L + 2, Unit{});
  for (int l = 0; l < L + 2; ++l) {
    Unit& u = pl.units[l];
    if (l < L) {
      u.cls = U_BLOCK;
      u.n = phi;
      u.owner = l % D;
      u.canon = V * H + static_cast<int64_t>(l) * phi;
      u.n_nd = 2;  // RMSNorm gains: no weight decay (R1)
      u.nd_lo[0] = 0;
      u.nd_hi[0] = H;
      u.nd_lo[1] = H + 4 * H * H;
      u.nd_hi[1] = 2 * H + 4 * H * H;
    } else if (l == L) {
      u.cls = U_E;
      u.n = V * H;
      u.owner = 0;
      u.canon = 0;
    } else {
      u.cls = U_F;
      u.n = H + V * H;
      u.owner = D - 1;
      u.canon = V * H + static_cast<int64_t>(L) * phi;
      u.n_nd = 1;
      u.nd_lo[0] = 0;
      u.nd_hi[0] = H;
    }
    if (literal) {
      // device i of group k holds W_{(D·i+k) mod P}; layer l (L mod P = 0) is shard l mod P, i.e.
      // group l mod D, member (l / D) mod G -- the rail counterpart of every group (R7).  E: device 0, F: P − 1.
      u.hold = l < L ? (l / D) % G : (l == L ? 0 : G - 1);
      u.n_pad = pad_to(u.n, 1);
      u.s = u.n_pad;
      u.owned = (u.owner == k && u.hold == j);
      u.lo = 0;
    } else {
      u.n_pad = pad_to(u.n, G);
      u.s = u.n_pad / G;
      u.owned = (u.owner == k);
      u.lo = static_cast<int64_t>(j) * u.s;
    }
    pl.max_pad = std::max(pl.max_pad, u.n_pad);
    pl.max_s = std::max(pl.max_s, u.s);
  }
  for (int l = 0; l < L + 2; ++l)  // canonical shard order: layers ascending, then E, then F
    if (pl.units[l].owned) {
      pl.units[l].off = pl.owned_total;
      pl.owned_total += pl.units[l].s;
    }
  return pl;
}

// Map every rank's weight / gradient buffers (COLLECTIVE); on success the step uses the peer path
void setup_p2p() {
  Ctx& c = *g;
  const char* e = std::getenv("TAWPIPE_COMM");
  if (c.world == 1 || c.ring || c.literal || (e && std::string(e) == "nccl")) return;
  TP_CHECK(c.P <= kSigRanks && c.G <= kMaxPartialSources && c.G - 1 + c.D - 1 <= kMaxSignalTargets && c.G * 1 + c.D <= 16,
           TAWPIPE_ECONFIG, "peer path: at most 64 ranks, 8 members per group, 16 gradient sources");
  c.sig = static_cast<uint32_t*>(dmalloc(SK_N * kSigRanks * sizeof(uint32_t)));
  c.sig_expect.assign(static_cast<size_t>(SK_N) * kSigRanks, 0);
  TP_CUDA(cudaMemsetAsync(c.sig, 0, SK_N * kSigRanks * sizeof(uint32_t), c.cs));
  if (c.D > 1) c.part = dmalloc(4 * c.max_s * c.esz);
  std::vector<void*> local(PB_N, nullptr);
  local[PB_WIRE] = c.wire;
  local[PB_WBUF0] = c.wbuf[0];
  local[PB_WBUF1] = c.wbuf[1];
  local[PB_EBUF] = c.ebuf;
  local[PB_FBUF] = c.fbuf;
  local[PB_GACC0] = c.gacc[0];
  local[PB_GACC1] = c.gacc[1];
  local[PB_GACCE] = c.gaccE;
  local[PB_GACCF] = c.gaccF;
  local[PB_PART] = c.part;
  local[PB_SIG] = c.sig;
  TP_CUDA(cudaStreamSynchronize(c.cs));
  c.p2p = peer_open(c.world_comm, c.rank, c.world, local, c.peer, c.cs);
  c.gofs.assign(static_cast<size_t>(c.D) * (c.L + 2), 0);
  for (int kk = 0; kk < c.D; ++kk) {
    Plan pl = make_plan(c.P, c.G, c.L, c.H, c.I, c.V, kk * c.G, false);
    for (int uid = 0; uid < c.L + 2; ++uid) c.gofs[static_cast<size_t>(kk) * (c.L + 2) + uid] = pl.units[uid].off;
  }
}

void build(int P, int G, int L, const tawpipe_dims* d, int N) {
  Ctx& c = *g;
  validate(P, G, L, d, N, c.world);
  const int D = P / G;
  c.P = P;
  c.G = G;
  c.D = D;
  c.k = c.rank / G;
  c.j = c.rank % G;
  c.L = L;
  c.N = N;
  c.m = N / P;
  c.dims = *d;
  c.H = d->hidden;
  c.nh = d->heads;
  c.dh = d->hidden / d->heads;
  c.I = d->ffn;
  c.V = d->vocab;
  c.S = d->seq;
  c.Bm = d->micro_bs;
  c.T = static_cast<int64_t>(c.Bm) * c.S;
  c.bf = d->dtype == TAWPIPE_BF16;
  c.ring = (d->schedule & TAWPIPE_RING) != 0;
  c.literal = (d->schedule & TAWPIPE_LITERAL) != 0;
  c.esz = c.bf ? 2 : 4;
  const int64_t H = c.H, I = c.I, V = c.V;
  c.phi = 4 * H * H + 3 * H * I + 2 * H;
  {
    Plan pl = make_plan(P, G, L, H, I, V, c.rank, (d->schedule & TAWPIPE_LITERAL) != 0);
    plan_ledger(pl, P, G, L, d->schedule, c.rank, c.ledger_plan);
    c.units = pl.units;
    c.owned_total = pl.owned_total;
    c.max_pad = pl.max_pad;
    c.max_s = pl.max_s;
  }
  // ---- streams, events, communicators
  TP_CUDA(cudaStreamCreateWithFlags(&c.cs, cudaStreamNonBlocking));
  TP_CUDA(cudaStreamCreateWithFlags(&c.ws, cudaStreamNonBlocking));
  {
    // the gradient stream runs at the highest priority, so its short, memory-bound reduction and AdamW blocks are
    // dispatched ahead of the compute stream's pending attention / GEMM blocks (C3, N = 4: the fused kernels' time
    // 186 -> 28 ms, step +0.3 %, same box A/B); TAWPIPE_GS_PRIORITY=0 restores the default priority
    const char* e = std::getenv("TAWPIPE_GS_PRIORITY");
    int lo = 0, hi = 0;
    TP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (!(e && std::atoi(e) == 0))
      TP_CUDA(cudaStreamCreateWithPriority(&c.gs, cudaStreamNonBlocking, hi));
    else
      TP_CUDA(cudaStreamCreateWithFlags(&c.gs, cudaStreamNonBlocking));
  }
  for (int i = 0; i < 2; ++i) {
    TP_CUDA(cudaEventCreateWithFlags(&c.w_ready[i], cudaEventDisableTiming));
    TP_CUDA(cudaEventCreateWithFlags(&c.w_free[i], cudaEventDisableTiming));
    TP_CUDA(cudaEventCreateWithFlags(&c.g_ready[i], cudaEventDisableTiming));
    TP_CUDA(cudaEventCreateWithFlags(&c.g_free[i], cudaEventDisableTiming));
  }
  for (cudaEvent_t* e : {&c.evE, &c.evF, &c.evGF, &c.evGE}) TP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&c.ev_s0, &c.ev_s1, &c.ev_ws0, &c.ev_ws1, &c.ev_gs0, &c.ev_gs1}) TP_CUDA(cudaEventCreate(e));
  if (c.world > 1) {
    // group communicator: color k, rank j ; rail communicator: color j, rank k (R5)
    TP_NCCL(ncclCommSplit(c.world_comm, c.k, c.j, &c.wg, nullptr));
    TP_NCCL(ncclCommSplit(c.world_comm, c.j, c.k, &c.wr, nullptr));
    TP_NCCL(ncclCommSplit(c.world_comm, c.k, c.j, &c.gg, nullptr));
    TP_NCCL(ncclCommSplit(c.world_comm, c.j, c.k, &c.gr, nullptr));
  }
  // ---- DBS state
  const size_t esz = c.esz;
  c.master = (float*)dmalloc(c.owned_total * 4);
  c.mom = (float*)dmalloc(c.owned_total * 4);
  c.vel = (float*)dmalloc(c.owned_total * 4);
  c.wire = dmalloc(c.owned_total * esz);
  TP_CUDA(cudaMemsetAsync(c.mom, 0, c.owned_total * 4, c.cs));
  TP_CUDA(cudaMemsetAsync(c.vel, 0, c.owned_total * 4, c.cs));
  const bool alias_layers = (G == 1 && D == 1);
  if (!alias_layers) {
    c.wbuf[0] = dmalloc(c.units[0].n_pad * esz);
    c.wbuf[1] = dmalloc(c.units[0].n_pad * esz);
  }
  if (!(G == 1 && c.units[L].owned)) c.ebuf = dmalloc(c.units[L].n_pad * esz);
  if (!(G == 1 && c.units[L + 1].owned)) c.fbuf = dmalloc(c.units[L + 1].n_pad * esz);
  c.gacc[0] = (float*)dmalloc(c.units[0].n_pad * 4);
  c.gacc[1] = (float*)dmalloc(c.units[0].n_pad * 4);
  c.gaccE = (float*)dmalloc(c.units[L].n_pad * 4);
  c.gaccF = (float*)dmalloc(c.units[L + 1].n_pad * 4);
  TP_CUDA(cudaMemsetAsync(c.gacc[0], 0, c.units[0].n_pad * 4, c.cs));
  TP_CUDA(cudaMemsetAsync(c.gacc[1], 0, c.units[0].n_pad * 4, c.cs));
  TP_CUDA(cudaMemsetAsync(c.gaccF, 0, c.units[L + 1].n_pad * 4, c.cs));   // padding stays zero (nothing writes it)
  c.dg_scratch = (float*)dmalloc(rmsnorm_bwd_scratch_floats(c.T, c.H) * 4);
  if (G > 1 || D > 1) c.gwire = dmalloc(c.max_pad * esz);
  if (G > 1) c.rsout = dmalloc(c.max_s * esz);
  if (D > 1) c.crecv = dmalloc(c.max_s * (D - 1) * esz);
  setup_p2p();   // NVLink peer mappings (GWPS on one box); NCCL collectives otherwise
  // ---- activations
  const int64_t T = c.T;
  const int m = c.m;
  c.ck.resize(static_cast<size_t>(L + 1) * m);
  for (auto& p : c.ck) p = dmalloc(T * H * esz);
  const size_t n_acts = d->ckpt ? 1 : static_cast<size_t>(L) * m;
  c.acts.resize(n_acts);
  for (auto& A : c.acts) {
    A.a = dmalloc(T * H * esz);
    A.qkv = dmalloc(T * 3 * H * esz);
    A.o = dmalloc(T * H * esz);
    A.h1 = dmalloc(T * H * esz);
    A.b = dmalloc(T * H * esz);
    A.gu = dmalloc(T * 2 * I * esz);
    A.y = dmalloc(T * I * esz);
    A.r1 = (float*)dmalloc(T * 4);
    A.r2 = (float*)dmalloc(T * 4);
    A.lse = (float*)dmalloc(T * c.nh * 4);
  }
  c.dhb.resize(m);
  for (auto& p : c.dhb) p = dmalloc(T * H * esz);
  if (!c.bf || gemm_force_simt()) c.dY = dmalloc(T * I * esz);   // the tcgen05 path fuses SwiGLU' into the dgrad
  c.dGU = dmalloc(T * 2 * I * esz);
  c.db = dmalloc(T * H * esz);
  c.dh1 = dmalloc(T * H * esz);
  c.dO = dmalloc(T * H * esz);
  c.dqkv = dmalloc(T * 3 * H * esz);
  c.da = dmalloc(T * H * esz);
  c.delta = (float*)dmalloc(2 * T * c.nh * 4);   // δ, then the log2-domain LSE of the tcgen05 backward
  c.dq_acc = c.bf ? (float*)dmalloc(T * H * 4) : nullptr;
  c.emb_scratch_bytes = embed_bwd_scratch_bytes(T);
  c.emb_scratch = dmalloc(c.emb_scratch_bytes);
  c.Tc = std::min<int64_t>(T, 8192);
  c.fnorm = dmalloc(T * H * esz);
  c.df = dmalloc(T * H * esz);
  c.logits = dmalloc(c.Tc * V * esz);
  c.rstd_f = (float*)dmalloc(T * 4);
  c.loss_rows = (float*)dmalloc(T * 4);
  c.d_loss = (double*)dmalloc(sizeof(double));
  TP_CUDA(cudaMallocHost(&c.h_loss, sizeof(double)));
  const int64_t tok_elems = static_cast<int64_t>(m) * c.Bm * (c.S + 1);
  c.d_tok = (int32_t*)dmalloc(tok_elems * 4);
  c.d_in = (int32_t*)dmalloc(static_cast<int64_t>(m) * T * 4);
  c.d_tgt = (int32_t*)dmalloc(static_cast<int64_t>(m) * T * 4);
  TP_CUDA(cudaMallocHost(&c.h_tok, tok_elems * 4));
  // RoPE tables in fp64 on the host, stored fp32 (R13)
  {
    std::vector<float> cs, sn;
    rope_tables_host(c.S, c.dh, d->rope_theta, cs, sn);
    c.cosT = (float*)dmalloc(cs.size() * 4);
    c.sinT = (float*)dmalloc(sn.size() * 4);
    TP_CUDA(cudaMemcpyAsync(c.cosT, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, c.cs));
    TP_CUDA(cudaMemcpyAsync(c.sinT, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice, c.cs));
    if (c.bf && !gemm_force_simt() && (2 * c.H) % 256 == 0 && c.dh % 64 == 0) {
      const int half = c.dh / 2;
      std::vector<float> both(static_cast<size_t>(c.S) * c.dh);
      for (int p = 0; p < c.S; ++p)
        for (int i = 0; i < half; ++i) {
          both[static_cast<size_t>(p) * c.dh + i] = cs[static_cast<size_t>(p) * half + i];
          both[static_cast<size_t>(p) * c.dh + half + i] = sn[static_cast<size_t>(p) * half + i];
        }
      c.rope_cs = (float*)dmalloc(both.size() * 4);
      TP_CUDA(cudaMemcpyAsync(c.rope_cs, both.data(), both.size() * 4, cudaMemcpyHostToDevice, c.cs));
    }
    TP_CUDA(cudaStreamSynchronize(c.cs));
  }
  // ---- selective checkpointing (ckpt = 1): keep activations level by level while device memory allows
  if (d->ckpt == 1) {
    size_t fr = 0, tot = 0;
    TP_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t margin = size_t(P > 1 ? 6 : 3) << 30;   // NCCL channels (none at P = 1), allocator slack
    size_t budget = fr > margin ? fr - margin : 0;
    if (const char* e = std::getenv("TAWPIPE_KEEP_BUDGET_KB")) budget = std::min(budget, size_t(std::atoll(e)) << 10);
    const size_t n = static_cast<size_t>(L) * m, TT = static_cast<size_t>(T);
    const size_t cost[4] = {TT * H * esz + TT * c.nh * 4, TT * 3 * H * esz, TT * H * esz, TT * 2 * I * esz};
    c.kept.assign(n, Kept{});
    for (int lv = 0; lv < 4; ++lv) {
      const size_t cnt = std::min(n, budget / cost[lv]);
      for (size_t i = 0; i < cnt; ++i) {
        Kept& k = c.kept[i];
        switch (lv) {
          case 0: k.o = dmalloc(TT * H * esz); k.lse = (float*)dmalloc(TT * c.nh * 4); break;
          case 1: k.qkv = dmalloc(TT * 3 * H * esz); break;
          case 2: k.h1 = dmalloc(TT * H * esz); break;
          case 3: k.gu = dmalloc(TT * 2 * I * esz); break;
        }
        k.flags |= static_cast<uint8_t>(1u << lv);
      }
      budget -= cnt * cost[lv];
      if (cnt < n) break;
    }
  }
  // ---- seeded device-side initialisation of the owned stripes (R20)
  for (int l = 0; l < L + 2; ++l) {
    const Unit& u = c.units[l];
    if (!u.owned) continue;
    const int64_t lo = u.lo;  // owned piece's start in unit coordinates
    float* ms = c.master + u.off;
    BY_TYPE(init_normal<float>((float*)wptr(c.wire, u.off), ms, u.s, u.canon + lo, d->seed, 0.02f, c.cs),
            init_normal<bf16>((bf16*)wptr(c.wire, u.off), ms, u.s, u.canon + lo, d->seed, 0.02f, c.cs));
    for (int r = 0; r < u.n_nd; ++r) {  // gains = 1
      const int64_t a = std::max(u.nd_lo[r], lo), b = std::min(u.nd_hi[r], lo + u.s);
      if (a < b) fill_f32(ms + (a - lo), b - a, 1.0f, c.cs);
    }
    if (u.n < lo + u.s) {  // zero padding
      const int64_t a = std::max(u.n, lo);
      fill_f32(ms + (a - lo), lo + u.s - a, 0.0f, c.cs);
    }
    BY_TYPE(cast_f32<float>(ms, (float*)wptr(c.wire, u.off), u.s, c.cs),
            cast_f32<bf16>(ms, (bf16*)wptr(c.wire, u.off), u.s, c.cs));
  }
  TP_CUDA(cudaStreamSynchronize(c.cs));
  c.barrier_buf = dmalloc(sizeof(int));
  TP_CUDA(cudaMemset(c.barrier_buf, 0, sizeof(int)));
  world_barrier();   // every owner's wire copy is initialised before any peer can pull it
  c.inited = true;
}

void load(const float* full, int64_t n) {
  Ctx& c = *g;
  const int64_t expect = 2 * static_cast<int64_t>(c.V) * c.H + static_cast<int64_t>(c.L) * c.phi + c.H;
  TP_CHECK(n == expect, TAWPIPE_ECONFIG, "tawpipe_load: expected " + std::to_string(expect) + " elements, got " +
                                             std::to_string(n));
  for (int l = 0; l < c.L + 2; ++l) {
    const Unit& u = c.units[l];
    if (!u.owned) continue;
    const int64_t lo = u.lo;
    float* ms = c.master + u.off;
    // every copy is ordered on c.cs: the compute stream is non-blocking and would not see legacy-stream copies
    TP_CUDA(cudaMemsetAsync(ms, 0, u.s * 4, c.cs));
    const int64_t valid = std::max<int64_t>(0, std::min(u.n, lo + u.s) - lo);
    if (valid > 0) TP_CUDA(cudaMemcpyAsync(ms, full + u.canon + lo, valid * 4, cudaMemcpyHostToDevice, c.cs));
    BY_TYPE(cast_f32<float>(ms, (float*)wptr(c.wire, u.off), u.s, c.cs),
            cast_f32<bf16>(ms, (bf16*)wptr(c.wire, u.off), u.s, c.cs));
  }
  TP_CUDA(cudaMemsetAsync(c.mom, 0, c.owned_total * 4, c.cs));
  TP_CUDA(cudaMemsetAsync(c.vel, 0, c.owned_total * 4, c.cs));
  TP_CUDA(cudaStreamSynchronize(c.cs));
  world_barrier();   // no peer pulls a wire copy this rank is still rewriting
  c.step_t = 0;
}

void destroy() {
  if (!g) return;
  cudaDeviceSynchronize();
  if (!g->peer.empty()) peer_close(g->peer, g->rank);
  for (void* p : g->allocs) cudaFree(p);
  if (g->h_tok) cudaFreeHost(g->h_tok);
  if (g->h_loss) cudaFreeHost(g->h_loss);
  for (ncclComm_t cm : {g->wg, g->wr, g->gg, g->gr})
    if (cm) ncclCommDestroy(cm);
  if (g->world_comm) ncclCommDestroy(g->world_comm);
  for (cudaEvent_t e : g->ev_pool) cudaEventDestroy(e);
  if (g->inited) {   // the named events build() created
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t e : {g->w_ready[i], g->w_free[i], g->g_ready[i], g->g_free[i]}) cudaEventDestroy(e);
    for (cudaEvent_t e : {g->evE, g->evF, g->evGF, g->evGE, g->ev_s0, g->ev_s1, g->ev_ws0, g->ev_ws1, g->ev_gs0,
                          g->ev_gs1})
      cudaEventDestroy(e);
  }
  if (g->cs) cudaStreamDestroy(g->cs);
  if (g->ws) cudaStreamDestroy(g->ws);
  if (g->gs) cudaStreamDestroy(g->gs);
  delete g;
  g = nullptr;
}

}  // namespace
}  // namespace tp

using namespace tp;

extern "C" {

int tawpipe_get_unique_id(void* out) {
  return guarded([&] {
    TP_CHECK(out, TAWPIPE_ECONFIG, "out is NULL");
    ncclUniqueId id;
    TP_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

int tawpipe_bootstrap(int rank, int world, int device, const void* uid) {
  return guarded([&] {
    TP_CHECK(world >= 1 && rank >= 0 && rank < world, TAWPIPE_ECONFIG, "bad rank/world");
    if (g) destroy();
    g = new Ctx();
    g->rank = rank;
    g->world = world;
    g->device = device;
    TP_CUDA(cudaSetDevice(device));
    if (world > 1) {
      TP_CHECK(uid, TAWPIPE_ECONFIG, "unique_id required when world > 1");
      ncclUniqueId id;
      std::memcpy(&id, uid, sizeof(id));
      TP_NCCL(ncclCommInitRank(&g->world_comm, world, id, rank));
    }
    g->booted = true;
  });
}

int tawpipe_plan(int n_devices, int group_size, int n_layers, const tawpipe_dims* dims, int n_micro, int rank,
                 uint64_t* ledger_out, int64_t* shard_elems_out) {
  return guarded([&] {
    validate(n_devices, group_size, n_layers, dims, n_micro, n_devices);
    TP_CHECK(rank >= 0 && rank < n_devices, TAWPIPE_ECONFIG, "rank out of range");
    const bool literal = (dims->schedule & TAWPIPE_LITERAL) != 0;
    Plan pl = make_plan(n_devices, group_size, n_layers, dims->hidden, dims->ffn, dims->vocab, rank, literal);
    uint64_t led[TAWPIPE_LEDGER_N] = {};
    plan_ledger(pl, n_devices, group_size, n_layers, dims->schedule, rank, led);
    if (ledger_out) std::memcpy(ledger_out, led, sizeof(led));
    if (shard_elems_out) *shard_elems_out = pl.owned_total;
  });
}

int tawpipe_init(int n_devices, int group_size, int n_layers, const tawpipe_dims* dims, int n_micro) {
  if (!g || !g->booted) {
    g_err = "tawpipe_init before tawpipe_bootstrap";
    return TAWPIPE_EUNINIT;
  }
  if (g->inited) {
    g_err = "already initialised; call tawpipe_finalize first";
    return TAWPIPE_ECONFIG;
  }
  return guarded([&] { build(n_devices, group_size, n_layers, dims, n_micro); });
}

int tawpipe_load(const float* full, int64_t n) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  return guarded([&] {
    TP_CHECK(full, TAWPIPE_ECONFIG, "full_model is NULL");
    load(full, n);
  });
}

static float step_common(const int32_t* tok, bool dev) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return NAN;
  }
  double loss = NAN;
  int rc = guarded([&] {
    TP_CHECK(tok, TAWPIPE_ECONFIG, "tokens is NULL");
    loss = run_step(tok, dev);
  });
  return rc == TAWPIPE_OK ? static_cast<float>(loss) : NAN;
}

float tawpipe_step(const int32_t* tokens) { return step_common(tokens, false); }
float tawpipe_step_device(const int32_t* dev_tokens) { return step_common(dev_tokens, true); }

int64_t tawpipe_shard_elems(void) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  return g->owned_total;
}

int64_t tawpipe_shard(float* out) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  int rc = guarded([&] {
    TP_CHECK(out, TAWPIPE_ECONFIG, "out is NULL");
    TP_CUDA(cudaDeviceSynchronize());
    TP_CUDA(cudaMemcpy(out, g->master, g->owned_total * 4, cudaMemcpyDeviceToHost));
  });
  return rc == TAWPIPE_OK ? g->owned_total : rc;
}

int tawpipe_ledger(uint64_t* out, int n) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  if (!out || n < TAWPIPE_LEDGER_N) {
    g_err = "ledger buffer too small";
    return TAWPIPE_ECONFIG;
  }
  std::memcpy(out, g->ledger, sizeof(g->ledger));
  return TAWPIPE_OK;
}

int tawpipe_stats(double* out, int n) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  if (!out || n < TAWPIPE_STATS_N) {
    g_err = "stats buffer too small";
    return TAWPIPE_ECONFIG;
  }
  std::memcpy(out, g->stats, sizeof(g->stats));
  return TAWPIPE_OK;
}

int tawpipe_set_timing(int on) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  g->timing = on != 0;
  return TAWPIPE_OK;
}

int64_t tawpipe_trace_json(char* out, int64_t cap) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  const int64_t n = static_cast<int64_t>(g->trace_json.size());
  if (out != nullptr && cap > 0) {
    const int64_t k = std::min<int64_t>(n, cap - 1);
    std::memcpy(out, g->trace_json.data(), static_cast<size_t>(k));
    out[k] = 0;
  }
  return n;
}

int tawpipe_set_link_emulation(double inter_gbps, double latency_us, int node_size) {
  if (!g || !g->inited) {
    g_err = "not initialised";
    return TAWPIPE_EUNINIT;
  }
  if (!(inter_gbps >= 0) || !(latency_us >= 0) || node_size < 0 || (node_size > 0 && g->P % node_size != 0)) {
    g_err = "link emulation: need inter_gbps >= 0, latency_us >= 0, node_size >= 0 dividing n_devices";
    return TAWPIPE_ECONFIG;
  }
  g->emu_gbps = inter_gbps;
  g->emu_lat_us = latency_us;
  g->emu_node = node_size;
  return TAWPIPE_OK;
}

const char* tawpipe_last_error(void) { return g_err.c_str(); }

void tawpipe_finalize(void) { destroy(); }

}  // extern "C"
