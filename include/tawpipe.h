/*
 * tawpipe.h -- C ABI of the B200-native TawPipe training-step library (libtawpipe.so).
 *
 * What the library computes.  One synchronous training iteration of a LLaMA-style
 * decoder under TawPipe's three mechanisms (§3.1):
 *   - DBS, device-bound storage: every layer's weights, gradients and optimizer state are
 *     statically bound to devices (§3.2).  Reading R6: layer l is
 *     owned by group l mod D and striped G ways over the group's members.
 *   - GWPS, group-based weight pipeline scheduling: devices form D contiguous groups of G
 *     (§3.3); weights move by intra-group all-gather and inter-group rail P2P,
 *     gradients by intra-group reduce-scatter and rail P2P to the owner.
 *   - CCO, communication-computation overlap: layer l+1 is prefetched on a side stream
 *     while layer l computes (§3.4).
 * The result equals one step of plain single-device mini-batch AdamW on all N·B sequences
 * (SURVEY.md §8(c)); parity is checked against the fp64 oracle in oracle/.
 *
 * Process model.  SPMD, one process per GPU, one live context per process.  Calls marked
 * COLLECTIVE must be made by every rank in the same order.  Calls are not thread-safe.
 *
 * Errors.  Functions returning int return TAWPIPE_OK (0) or a negative code; tawpipe_step
 * returns NaN on error.  tawpipe_last_error() describes the last failure.  After any error
 * other than TAWPIPE_ECONFIG the context is unusable until tawpipe_finalize().
 *
 * There is no CPU fallback: every step of the path runs in this library's CUDA kernels.
 */
#ifndef TAWPIPE_H_
#define TAWPIPE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TAWPIPE_OK          0
#define TAWPIPE_ECONFIG    -2   /* invalid configuration / argument (SPEC.md:515 exit code 2)        */
#define TAWPIPE_EINVARIANT -3   /* internal invariant failure (SPEC.md:515 exit code 3): a layer slot   *
                                 * about to be computed on does not carry the version tag (unit, step)  *
                                 * of that layer, or -- end-of-step check of the NVLink peer path -- a  *
                                 * sequence flag a peer wrote does not end at the value the schedule    *
                                 * implies (a lost, duplicated or mis-numbered signal), or the step's   *
                                 * byte ledger differs from the planned schedule's (tawpipe_plan)       */
#define TAWPIPE_ERUNTIME   -4   /* CUDA or NCCL runtime error (SPEC.md:515 exit code 4)              */
#define TAWPIPE_EUNINIT    -5   /* call before tawpipe_bootstrap / tawpipe_init                       */

#define TAWPIPE_FP32 0          /* parity path: every tensor, wire and accumulator fp32 (SIMT FMA)    */
#define TAWPIPE_BF16 1          /* bf16 weights/activations/wire, fp32 accumulation/master/m/v        */

/* schedule flags (tawpipe_dims.schedule) */
#define TAWPIPE_GWPS   0        /* default: the paper's schedule                                     */
#define TAWPIPE_NO_CCO 1        /* ablation: gather of layer l+1 waits for compute of l */
#define TAWPIPE_RING   2        /* WeiPipe-style ring (also the paper's "w/o GWPS"
                                   ablation): whole layers owned by device l mod P (needs
                                   group_size 1); weights hop owner -> owner+1 -> ... around the ring,
                                   gradients accumulate hop by hop from owner+1 and end at the owner.
                                   The FSDP-style global schedule is group_size = n_devices (D = 1).     */
#define TAWPIPE_LITERAL 4       /* paper-literal collectives (NEXT-2): whole
                                   layers, device i of group k owns W_{(D·i+k) mod P} (layer l is shard
                                   l mod P; needs L mod P = 0), E on device 0, F on device P−1.  Gather:
                                   owner -> rail counterpart (k, i) of every other group (P2P), then
                                   ncclBroadcast from (k, i) inside each group; reduction: ncclReduce to
                                   (k, i) in each group, then P2P to the owner, which sums the D group
                                   contributions and applies AdamW.  tawpipe_shard returns whole owned
                                   units.  Exclusive with TAWPIPE_RING; combinable with TAWPIPE_NO_CCO.  */

#define TAWPIPE_LEDGER_N 24     /* see tawpipe_ledger */
#define TAWPIPE_STATS_N  19     /* see tawpipe_stats  */

/* Model dimensions and hyper-parameters.  Symbols follow PAPER.md Table 1;
 * the rest are LLaMA-2 conventions. */
typedef struct tawpipe_dims {
  int32_t hidden;        /* H                                                                   */
  int32_t heads;         /* n_h; head dim d_h = H / n_h                                          */
  int32_t ffn;           /* I, SwiGLU width                                                      */
  int32_t vocab;         /* V                                                                    */
  int32_t seq;           /* S, tokens per sequence fed to the model                              */
  int32_t micro_bs;      /* B, sequences per micro-batch                                          */
  int32_t dtype;         /* TAWPIPE_FP32 | TAWPIPE_BF16                                          */
  int32_t ckpt;          /* activation checkpointing: 0 none (all activations kept);
                          * 1 keep each layer's input h_l and recompute the layer in backward, but
                          * keep more of it while device memory allows (selective: attention O+LSE,
                          * then q|k|v, then h1, then the MLP's gu, per (layer, micro-batch); the
                          * recompute skips what was kept; results are bit-identical except the
                          * MLP's y, re-derived from the kept bf16 gu: one bf16 rounding apart);
                          * 2 keep h_l only (full recompute)                                      */
  int32_t schedule;      /* TAWPIPE_GWPS, TAWPIPE_RING or TAWPIPE_LITERAL, optionally | TAWPIPE_NO_CCO */
  int32_t reserved;      /* must be 0                                                            */
  float lr, beta1, beta2, adam_eps, weight_decay;   /* AdamW, torch semantics (R1)               */
  float rms_eps, rope_theta;                        /* 1e-5, 10000 (R10)                          */
  uint64_t seed;         /* device-side N(0,0.02) init when tawpipe_load is not called (R20)    */
} tawpipe_dims;

/* Create an NCCL unique id (128 bytes) on the calling rank (rank 0 of the job).  LOCAL.
 * out: caller-owned buffer of >= 128 bytes.  Returns 0 or TAWPIPE_ERUNTIME. */
int tawpipe_get_unique_id(void* out);

/* Bind this process to `device` and, when world > 1, create the world NCCL communicator from
 * `unique_id` (128 bytes from tawpipe_get_unique_id on rank 0, distributed by the caller --
 * the Python binding uses torch.distributed for that).  COLLECTIVE when world > 1.
 * unique_id may be NULL when world == 1. */
int tawpipe_bootstrap(int rank, int world, int device, const void* unique_id);

/* Build the DBS plan and allocate all device state.  COLLECTIVE.
 *   n_devices  P; must equal the bootstrap world size.
 *   group_size G = P / D; P mod G == 0 ("P mod D = 0").
 *   n_layers   L; L mod D == 0 (reading R6 replaces the paper's L mod P = 0).
 *   dims       model dimensions (copied).
 *   n_micro    N micro-batches per iteration, N mod P == 0; each device takes m = N/P
 *              contiguous micro-batches (R4).
 * bf16 path shape limits: d_h in {64,128}, S mod 128 == 0, H, I, V multiples of 128.
 * Weights are initialised on the device from dims->seed; call tawpipe_load to override.
 * Returns 0, TAWPIPE_ECONFIG (message names the violated constraint) or TAWPIPE_ERUNTIME. */
int tawpipe_init(int n_devices, int group_size, int n_layers, const tawpipe_dims* dims, int n_micro);

/* Host-only dry run of the DBS plan for device `rank` (no GPU, no communication): validates the
 * configuration exactly like tawpipe_init (world size taken = n_devices), and returns the byte ledger one
 * tawpipe_step would record on that rank (same order as tawpipe_ledger; NULL to skip) and the number of
 * elements tawpipe_shard would write (NULL to skip).  The ledger is produced by the same accounting code
 * the real communication calls use.  LOCAL.  Returns 0 or TAWPIPE_ECONFIG. */
int tawpipe_plan(int n_devices, int group_size, int n_layers, const tawpipe_dims* dims, int n_micro, int rank,
                 uint64_t* ledger_out, int64_t* shard_elems_out);

/* Load the full model (host fp32, canonical layout, n_elems = V·H + L·φ + H + V·H with
 * φ = 4H²+3HI+2H): [E | layer 0 .. layer L−1 | γ_f | W_head], each layer
 * [attn_norm | Wq | Wk | Wv | Wo | mlp_norm | Wgate | Wup | Wdown], matrices row-major
 * [out, in].  Each rank keeps only its owned stripes; resets AdamW state and step count.
 * COLLECTIVE (no communication, but every rank must call it). */
int tawpipe_load(const float* full_model_fp32, int64_t n_elems);

/* One training iteration.  tokens: host int32 [N][B][S+1], identical on every rank; inputs are
 * positions 0..S−1 and targets 1..S of each sequence (R3).  The library copies this rank's
 * micro-batches to the device inside the call.  Returns the global mean loss over N·B·S
 * predicted tokens (R2), identical on all ranks, after every AdamW of the step has completed
 * (synchronous).  NaN on error.  COLLECTIVE. */
float tawpipe_step(const int32_t* tokens);

/* Same as tawpipe_step but `dev_tokens` is this rank's own slice, already resident in device
 * memory: int32 [m][B][S+1] with m = N/P.  Used to time the step with inputs in HBM. */
float tawpipe_step_device(const int32_t* dev_tokens);

/* Number of fp32 elements tawpipe_shard writes on this rank.  LOCAL. */
int64_t tawpipe_shard_elems(void);

/* Copy this rank's owned fp32 master stripes to host memory `out` (caller-owned, >=
 * tawpipe_shard_elems() floats), canonical order: owned decoder layers ascending, then E (if
 * owned), then F (if owned); for each unit, the stripe [j·s, (j+1)·s) of its zero-padded
 * flat vector (padding to G·64·ceil(n/(G·64)) elements).  Returns elements written or < 0. LOCAL. */
int64_t tawpipe_shard(float* out);

/* Byte ledger of the last step (logical elements): out[i] for
 * i = ((kind·2 + cls)·2 + dir)·3 + unit, kind {0 weight, 1 grad}, cls {0 intra-group,
 * 1 inter-group}, dir {0 received, 1 sent}, unit {0 decoder blocks, 1 E, 2 F}.
 * n >= TAWPIPE_LEDGER_N.  Bytes = elements × wire size (2 bf16, 4 fp32).  LOCAL. */
int tawpipe_ledger(uint64_t* out, int n);

/* Timing of the last step (requires tawpipe_set_timing(1) before it), n >= TAWPIPE_STATS_N:
 *  [0] step ms (compute stream, event to event)      [1] exposed-comm ms (compute-stream waits)
 *  [2] weight-comm ms (sum of gather P2P+all-gather) [3] grad-comm ms (sum of reduce-scatter + P2P)
 *  [4] GEMM ms (sum of tcgen05/SIMT GEMM launches)   [5] GEMM algorithmic GFLOP
 *  [6] GEMM launches                                 [7] attention ms   [8] attention GFLOP
 *  [9] AdamW ms   [10] AdamW algorithmic GB          [11] kernel launches in the step
 *  [12] peak device bytes allocated (GB)             [13] wire bytes per element
 *  [14] elementwise/norm ms
 *  [15] algorithmic GFLOP of the recompute passes (checkpointing) executed in the step
 *  [1] includes every compute-stream wait on peers and the step's tail (side-stream join + loss all-reduce)
 *  [16] 1 if the step ran the NVLink peer path (IPC-mapped copies / peer loads), 0 for NCCL collectives
 *  [17] GB of weight stripes this rank pulled over NVLink   [18] GB of gradients this rank's kernels read
 *       over NVLink (fp32 group stripes + wire-dtype rail partials)                                LOCAL. */
int tawpipe_stats(double* out, int n);

/* Enable (1) / disable (0) per-kernel CUDA-event timing for tawpipe_stats.  LOCAL. */
int tawpipe_set_timing(int on);

/* Trace-Event JSON (chrome://tracing / Perfetto) of the last step run with timing on (NEXT-4):
 * "X" events {name: gemm | attention | adamw | exposed_comm_wait | elementwise | weight_comm | grad_comm,
 * ts/dur in µs from the step's first compute-stream event, pid = rank, tid = stream (0 compute, 1 weights,
 * 2 gradients), args.work = algorithmic FLOP or bytes}; otherData = {rank, step, step_ms, busy_ms[3] (union of
 * each stream's regions), exposed_comm_ms, compute_idle_frac (compute stream neither computing nor waiting on
 * communication)}.  Writes min(length, cap − 1) bytes plus a NUL to `out` (caller-owned; may be NULL to query the
 * size) and returns the full length (0 before a timed step), or < 0 on error.  LOCAL. */
int64_t tawpipe_trace_json(char* out, int64_t cap);

/* Emulated link hierarchy (NEXT-3): devices are grouped into emulated nodes of `node_size`
 * consecutive ranks (0: the schedule's group size G).  Every weight / gradient transfer that crosses a node
 * boundary is followed on each participating stream by a device-side delay of latency_us + bytes / inter_gbps
 * (bytes: what the busiest endpoint moves across the boundary in that exchange: (D−1) stripes for the rail
 * exchange, (G−1) stripes for a cross-node ring all-gather / reduce-scatter, one unit per ring hop).  The paper's
 * testbed: 1.25 GB/s and 30 µs across nodes.  inter_gbps = 0 disables.  Results and the
 * ledger are unchanged.  Applies to later steps.  LOCAL (set the same values on every rank).  Returns 0 or
 * TAWPIPE_ECONFIG (negative values, node_size not dividing n_devices). */
int tawpipe_set_link_emulation(double inter_gbps, double latency_us, int node_size);

/* Thread-local description of the last error (never NULL).  LOCAL. */
const char* tawpipe_last_error(void);

/* Free all device memory and communicators.  COLLECTIVE when world > 1. */
void tawpipe_finalize(void);

/* ---- kernel-level entry points ------------------------------------------------------------------------------
 * Each runs exactly the kernel(s) tawpipe_step launches for that operation, on caller-owned DEVICE buffers of the
 * caller's current device, asynchronously on `stream` (cudaStream_t; NULL = legacy default stream) unless stated.
 * No context is needed.  Layouts are row-major; "dtype" is TAWPIPE_FP32 (fp32 tensors, SIMT kernels -- the fp32
 * parity path) or TAWPIPE_BF16 (bf16 tensors, fp32 arithmetic inside, tcgen05 where the op is a contraction).
 * Statistics (rstd, LSE, δ, loss rows) and accumulators are always fp32.  Return 0, TAWPIPE_ECONFIG (bad argument,
 * message in tawpipe_last_error) or TAWPIPE_ERUNTIME (CUDA launch error).  They serve the per-op parity tests.
 * Zero rows / tokens (RMSNorm, cross-entropy, embedding) are a no-op: nothing is launched or written. */

/* C[M,N] (+)= Σ_k A(m,k)·B(n,k) (the QKV/O/MLP/head projections and their dgrad/wgrad).
 * A(m,k) = A[m·a_ld + k] if a_kmajor else A[k·a_ld + m]; likewise B(n,k).
 * dtype: TAWPIPE_BF16 (bf16 A/B, tcgen05, fp32 accumulate in TMEM) or TAWPIPE_FP32 (SIMT).
 * c_f32: C is fp32 (else the dtype); accumulate: C += result (else C = result);
 * R (nullable, same dtype/ld as C): C = R + result.  bf16 shape limits: M mod 128, N mod 128,
 * K mod 64 == 0, 16-byte aligned pointers and leading dimensions. */
int tawpipe_gemm(int dtype, int64_t M, int64_t N, int64_t K,
                 const void* A, int64_t a_ld, int a_kmajor,
                 const void* B, int64_t b_ld, int b_kmajor,
                 void* C, int64_t c_ld, int c_f32, int accumulate,
                 const void* R, void* stream);

/* bf16 QKV projection with RoPE in the epilogue (the step's a5): qkv [M, N] = x·Wᵀ (x [M, K], W [N, K], both K-major),
 * then output columns [0, rope_cols) -- the q | k blocks, d_h-wide heads -- rotate-half rotated by p·θ_i with
 * p = row mod S and θ_i = theta^(−2i/d_h) (tables built as tawpipe_init builds them).  M, N mod 128, K mod 64,
 * d_h % 64 == 0, rope_cols % 256 == 0.  Synchronous. */
int tawpipe_gemm_rope(int64_t M, int64_t N, int64_t K, const void* x, const void* w, void* qkv, int S, int d_h,
                      float theta, int64_t rope_cols, void* stream);

/* bf16 gate/up projection with the SwiGLU forward in the epilogue (the step's a5 MLP):
 * [u | w] = x·W_guᵀ (x [M,K], W_gu [2I,K] = [W_gate ; W_up]); y [M,I] = SiLU(u)⊙w computed from the fp32
 * accumulators; gu [M,2I] (nullable) receives [u | w] in bf16.  M, 2I mod 256 or 128, K mod 64 == 0. */
int tawpipe_gemm_swiglu(int64_t M, int64_t I, int64_t K, const void* x, const void* w_gu, void* gu, void* y,
                        void* stream);

/* bf16 down-projection dgrad with the SwiGLU backward in the epilogue (the step's a7 MLP):
 * dY = dh·W_down (dh [M,K], W_down [K,I]), then dgu [M,2I] = [dY⊙w⊙σ(u)(1+u(1−σ(u))) | dY⊙SiLU(u)] with
 * u, w read from gu [M,2I] (SURVEY.md §8(c) SwiGLU backward); dY never reaches memory. */
int tawpipe_gemm_swiglu_bwd(int64_t M, int64_t I, int64_t K, const void* dh, const void* w_down, const void* gu,
                            void* dgu, void* stream);

/* Causal attention forward on one micro-batch: qkv [B·S, 3H] (q | k | v column blocks,
 * head h at columns h·d_h of each block, RoPE already applied), o [B·S, H], lse fp32 [B][n_h][S] (natural log).
 * bf16 tcgen05 path: S mod 128 == 0, d_h ∈ {64, 128} (else a SIMT kernel). */
int tawpipe_attention_fwd(int dtype, int B, int S, int n_h, int d_h,
                          const void* qkv, void* o, float* lse, void* stream);

/* Causal attention backward: do_ [B·S, H] -> dqkv [B·S, 3H] (dq | dk | dv, w.r.t. the roped q,k).
 * `scratch` is fp32 scratch of 2·B·n_h·S floats (δ = rowsum(dO⊙O) and the log2-domain LSE); `dq_acc` fp32
 * scratch of B·S·H floats (may be NULL for the fp32 path). */
int tawpipe_attention_bwd(int dtype, int B, int S, int n_h, int d_h,
                          const void* qkv, const void* o, const float* lse, const void* do_,
                          void* dqkv, float* scratch, float* dq_acc, void* stream);

/* Causal attention backward followed by the inverse RoPE of dq and dk (the step's order: dq, dk w.r.t. the UN-roped
 * q, k, rotated back by −p·θ_i with θ_i = theta^(−2i/d_h)); on the bf16 tcgen05 path the rotation is fused into the
 * kernel's dq conversion and dK epilogue, as in tawpipe_step.  Arguments as tawpipe_attention_bwd.  Synchronous. */
int tawpipe_attention_bwd_rope(int dtype, int B, int S, int n_h, int d_h, float theta,
                               const void* qkv, const void* o, const float* lse, const void* do_,
                               void* dqkv, float* scratch, float* dq_acc, void* stream);

/* RMSNorm forward: y[r] = x[r]·rstd[r]⊙γ, rstd[r] = (mean_H(x[r]²) + eps)^(−1/2);
 * x, y [rows, H] (dtype), γ [H] (dtype), rstd [rows] fp32. */
int tawpipe_rmsnorm_fwd(int dtype, int64_t rows, int H, const void* x, const void* gamma, float eps, void* y,
                        float* rstd, void* stream);

/* RMSNorm backward: dx = (res ? res : 0) + rstd·(dy⊙γ) − x·rstd³·mean_H(dy⊙γ⊙x) written to dx [rows, H];
 * dgamma_acc [H] fp32 += Σ_rows dy⊙x·rstd (accumulated, caller zeroes it; row-block partial sums added in block
 * order, so the result is bit-reproducible).  res nullable (the residual stream gradient added in the same pass). */
int tawpipe_rmsnorm_bwd(int dtype, int64_t rows, int H, const void* dy, const void* x, const void* gamma,
                        const float* rstd, const void* res, void* dx, float* dgamma_acc, void* stream);

/* Rotate-half RoPE in place on the q and k column blocks of qkv [B·S, 3·n_h·d_h]:
 * x'_i = x_i cos − x_{i+d/2} sin, x'_{i+d/2} = x_{i+d/2} cos + x_i sin with angle p·theta^(−2i/d_h), p = row mod S;
 * inverse != 0 rotates by −angle (the backward).  Tables are built in fp64 on the host, stored fp32, exactly as
 * tawpipe_init builds them.  Synchronous (returns after the kernel completed). */
int tawpipe_rope(int dtype, int B, int S, int n_h, int d_h, float theta, void* qkv, int inverse, void* stream);

/* SwiGLU forward: gu [rows, 2I] = [u | w] -> y [rows, I] = SiLU(u)⊙w (the SIMT / fp32 path's separate kernel). */
int tawpipe_swiglu_fwd(int dtype, int64_t rows, int I, const void* gu, void* y, void* stream);

/* SwiGLU backward: dy [rows, I], gu [rows, 2I] -> dgu [rows, 2I] = [dy⊙w⊙σ(u)(1+u(1−σ(u))) | dy⊙SiLU(u)]. */
int tawpipe_swiglu_bwd(int dtype, int64_t rows, int I, const void* dy, const void* gu, void* dgu, void* stream);

/* Fused cross-entropy forward + backward: logits [rows, V] are overwritten in place with
 * dz = (softmax(z) − onehot(target))·inv_denom; loss_rows [rows] fp32 = LSE(z) − z[target].  targets int32 [rows]
 * in [0, V). */
int tawpipe_cross_entropy(int dtype, int64_t rows, int V, void* logits, const int32_t* targets, float inv_denom,
                          float* loss_rows, void* stream);

/* Embedding forward: h[b·S + p] = E[tokens[b·tok_stride + p]], E [V, H], h [B·S, H]. */
int tawpipe_embed_fwd(int dtype, int B, int S, const int32_t* tokens, int64_t tok_stride, const void* E, int H,
                      void* h, void* stream);

/* Deterministic embedding backward: dE [V, H] fp32 += Σ_{p : token_p = v} dh[p] with each token's positions
 * summed in ascending order in fp32 (stable radix sort + segmented sum; bit-reproducible).  dh [B·S, H] (dtype).
 * Allocates its sort scratch stream-ordered on `stream`. */
int tawpipe_embed_bwd(int dtype, int B, int S, const int32_t* tokens, int64_t tok_stride, const void* dh, int H,
                      int V, float* dE, void* stream);

/* A non-owner group's rail partial (a8 on the NVLink peer path, "gradients are reduced within the
 * group, then sent to the owner"): out[i] = wire_dtype( Σ_{m = 0 .. n_src-1, in order} srcs[m][i] ), summed in fp32
 * (R16).  srcs [n_src] (1..8) device pointers of n fp32 elements each (in the step: the group members' fp32
 * gradient accumulators, read through IPC peer mappings); out [n] wire_dtype.  n % 4 == 0, pointers 16-byte
 * aligned.  n == 0 is a no-op. */
int tawpipe_group_partial(int wire_dtype, int n_src, const float* const* srcs, int64_t n, void* out, void* stream);

/* Fused gradient accumulation + AdamW on one owned stripe (a9; "updates ... applied at the owner";
 * AdamW torch semantics, R1):
 *   g = Σ_{groups gi ascending} ( Σ_{members, in order} srcs[·] )   in fp32 (R16),
 *   θ ← θ(1 − lr·wd) unless no-decay; m ← β1 m + (1−β1) g; v ← β2 v + (1−β2) g²;
 *   θ ← θ − lr·(m/(1−β1^step)) / (sqrt(v/(1−β2^step)) + eps);   wire ← wire_dtype(θ).
 * group_sizes [n_groups] (1..8 groups, 1..16 sources in total); srcs [Σ sizes] device pointers of n elements, each
 * fp32 if src_is_f32[i] else wire_dtype (any device memory the caller can address, including IPC-mapped peer
 * memory); master / m / v fp32 [n] and wire [n] updated in place.  no_decay (nullable) = {lo0, hi0, lo1, hi1}: element
 * i is not decayed if unit_off + i lies in [lo0, hi0) or [lo1, hi1).  hyper = {lr, β1, β2, eps, wd}; step >= 1. */
int tawpipe_adamw(int wire_dtype, int n_groups, const int* group_sizes, const void* const* srcs, const int* src_is_f32,
                  float* master, float* m, float* v, void* wire, int64_t n, int64_t unit_off,
                  const int64_t* no_decay, const float* hyper, int step, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TAWPIPE_H_ */
