"""Thin ctypes binding of libtawpipe.so (include/tawpipe.h).  Argument marshalling only: every step of the
training iteration runs in the library's CUDA kernels.  There is no CPU fallback -- if the library is
missing, importing this module's entry points raises.

Process model (SPMD, one process per GPU): ``bootstrap()`` reads RANK / WORLD_SIZE / LOCAL_RANK, creates
the NCCL unique id on rank 0 and distributes it through ``torch.distributed`` (PyTorch is used only for
that plumbing), then calls ``tawpipe_bootstrap``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtawpipe.so")

OK, ECONFIG, EINVARIANT, ERUNTIME, EUNINIT = 0, -2, -3, -4, -5
FP32, BF16 = 0, 1
GWPS, NO_CCO, RING, LITERAL = 0, 1, 2, 4
LEDGER_N, STATS_N = 24, 19

STATS_NAMES = ("step_ms", "exposed_comm_ms", "weight_comm_ms", "grad_comm_ms", "gemm_ms", "gemm_gflop",
               "gemm_launches", "attn_ms", "attn_gflop", "adamw_ms", "adamw_gb", "kernel_launches",
               "alloc_gb", "wire_bytes", "elementwise_ms", "recompute_gflop", "p2p", "nvlink_weight_gb",
               "nvlink_grad_gb")


class TawpipeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"tawpipe error {code}: {msg}")
        self.code = code


class Dims(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("heads", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("seq", ctypes.c_int32), ("micro_bs", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("ckpt", ctypes.c_int32), ("schedule", ctypes.c_int32),
                ("reserved", ctypes.c_int32),
                ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("adam_eps", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_float), ("seed", ctypes.c_uint64)]


_lib = None


def lib():
    """Load libtawpipe.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2511_09741_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
    sig = {
        "tawpipe_get_unique_id": (i32, [vp]),
        "tawpipe_bootstrap": (i32, [i32, i32, i32, vp]),
        "tawpipe_init": (i32, [i32, i32, i32, ctypes.POINTER(Dims), i32]),
        "tawpipe_plan": (i32, [i32, i32, i32, ctypes.POINTER(Dims), i32, i32, vp, vp]),
        "tawpipe_load": (i32, [vp, i64]),
        "tawpipe_step": (f32, [vp]),
        "tawpipe_step_device": (f32, [vp]),
        "tawpipe_shard_elems": (i64, []),
        "tawpipe_shard": (i64, [vp]),
        "tawpipe_ledger": (i32, [vp, i32]),
        "tawpipe_stats": (i32, [vp, i32]),
        "tawpipe_set_timing": (i32, [i32]),
        "tawpipe_trace_json": (i64, [vp, i64]),
        "tawpipe_set_link_emulation": (i32, [ctypes.c_double, ctypes.c_double, i32]),
        "tawpipe_last_error": (ctypes.c_char_p, []),
        "tawpipe_finalize": (None, []),
        "tawpipe_gemm": (i32, [i32, i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, i32, i32, vp, vp]),
        "tawpipe_attention_fwd": (i32, [i32, i32, i32, i32, i32, vp, vp, vp, vp]),
        "tawpipe_attention_bwd": (i32, [i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
        "tawpipe_attention_bwd_rope": (i32, [i32, i32, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp]),
        "tawpipe_gemm_rope": (i32, [i64, i64, i64, vp, vp, vp, i32, i32, f32, i64, vp]),
        "tawpipe_gemm_swiglu": (i32, [i64, i64, i64, vp, vp, vp, vp, vp]),
        "tawpipe_gemm_swiglu_bwd": (i32, [i64, i64, i64, vp, vp, vp, vp, vp]),
        "tawpipe_rmsnorm_fwd": (i32, [i32, i64, i32, vp, vp, f32, vp, vp, vp]),
        "tawpipe_rmsnorm_bwd": (i32, [i32, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
        "tawpipe_rope": (i32, [i32, i32, i32, i32, i32, f32, vp, i32, vp]),
        "tawpipe_swiglu_fwd": (i32, [i32, i64, i32, vp, vp, vp]),
        "tawpipe_swiglu_bwd": (i32, [i32, i64, i32, vp, vp, vp, vp]),
        "tawpipe_cross_entropy": (i32, [i32, i64, i32, vp, vp, f32, vp, vp]),
        "tawpipe_embed_fwd": (i32, [i32, i32, i32, vp, i64, vp, i32, vp, vp]),
        "tawpipe_embed_bwd": (i32, [i32, i32, i32, vp, i64, vp, i32, i32, vp, vp]),
        "tawpipe_group_partial": (i32, [i32, i32, vp, i64, vp, vp]),
        "tawpipe_adamw": (i32, [i32, i32, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp, vp, i32, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    return lib().tawpipe_last_error().decode()


def _check(rc):
    if rc != OK:
        raise TawpipeError(rc, last_error())
    return rc


# ---------------------------------------------------------------------------------------------- model layout
@dataclass
class ModelDims:
    n_layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    seq: int
    micro_bs: int = 1
    dtype: int = BF16
    ckpt: int = 0
    schedule: int = GWPS
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    weight_decay: float = 0.1
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0
    seed: int = 1234

    def to_c(self) -> Dims:
        return Dims(self.hidden, self.heads, self.ffn, self.vocab, self.seq, self.micro_bs, self.dtype, self.ckpt,
                    self.schedule, 0, self.lr, self.beta1, self.beta2, self.adam_eps, self.weight_decay,
                    self.rms_eps, self.rope_theta, self.seed)


_LAYER_ORDER = ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "w_gate", "w_up", "w_down")


def pack_full_model(params: dict) -> np.ndarray:
    """Canonical fp32 full-model vector for tawpipe_load: [E | layers | γ_f | W_head] (include/tawpipe.h)."""
    parts = [np.asarray(params["embed"], np.float32).ravel()]
    for lay in params["layers"]:
        parts += [np.asarray(lay[k], np.float32).ravel() for k in _LAYER_ORDER]
    parts += [np.asarray(params["final_norm"], np.float32).ravel(), np.asarray(params["head"], np.float32).ravel()]
    return np.ascontiguousarray(np.concatenate(parts))


# ---------------------------------------------------------------------------------------------- session
def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().tawpipe_get_unique_id(buf))
    return buf.raw


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def share_unique_id(rank: int, world: int, pg_backend: str = "gloo") -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts its 128 bytes to every rank."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group(backend=pg_backend, rank=rank, world_size=world)
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t = torch.tensor(list(unique_id()), dtype=torch.uint8)
    dist.broadcast(t, src=0)
    return bytes(t.tolist())


def bootstrap(rank=None, world=None, device=None, pg_backend="gloo"):
    """Bind to the GPU and build the world NCCL communicator.  For world > 1 the 128-byte NCCL unique id is
    broadcast from rank 0 with torch.distributed (plumbing only)."""
    r, w, loc = dist_env()
    rank = r if rank is None else rank
    world = w if world is None else world
    device = loc if device is None else device
    uid = share_unique_id(rank, world, pg_backend) if world > 1 else None
    buf = ctypes.create_string_buffer(uid, 128) if uid is not None else None
    _check(lib().tawpipe_bootstrap(rank, world, device, buf))
    return rank, world, device


class Session:
    """One TawPipe context: ``init`` (DBS plan + allocation), ``load``, ``step``, ``shard``, ``ledger``."""

    def __init__(self, n_devices: int, group_size: int, dims: ModelDims, n_micro: int):
        self.dims = dims
        self.P, self.G, self.N = n_devices, group_size, n_micro
        self._cdims = dims.to_c()
        _check(lib().tawpipe_init(n_devices, group_size, dims.n_layers, ctypes.byref(self._cdims), n_micro))

    def load(self, full: np.ndarray):
        full = np.ascontiguousarray(full, np.float32)
        _check(lib().tawpipe_load(full.ctypes.data, full.size))

    def step(self, tokens: np.ndarray) -> float:
        tokens = np.ascontiguousarray(tokens, np.int32)
        N, B, S1 = tokens.shape
        if N != self.N or B != self.dims.micro_bs or S1 != self.dims.seq + 1:
            raise TawpipeError(ECONFIG, f"tokens shape {tokens.shape} != ({self.N}, {self.dims.micro_bs}, "
                                        f"{self.dims.seq + 1})")
        loss = lib().tawpipe_step(tokens.ctypes.data)
        if loss != loss:
            raise TawpipeError(ERUNTIME, last_error())
        return loss

    def step_device(self, dev_ptr: int) -> float:
        loss = lib().tawpipe_step_device(ctypes.c_void_p(dev_ptr))
        if loss != loss:
            raise TawpipeError(ERUNTIME, last_error())
        return loss

    def shard(self) -> np.ndarray:
        n = lib().tawpipe_shard_elems()
        if n < 0:
            raise TawpipeError(n, last_error())
        out = np.empty(n, np.float32)
        r = lib().tawpipe_shard(out.ctypes.data)
        if r < 0:
            raise TawpipeError(r, last_error())
        return out

    def ledger(self) -> list:
        out = (ctypes.c_uint64 * LEDGER_N)()
        _check(lib().tawpipe_ledger(out, LEDGER_N))
        return [int(x) for x in out]

    def stats(self) -> dict:
        out = (ctypes.c_double * STATS_N)()
        _check(lib().tawpipe_stats(out, STATS_N))
        return dict(zip(STATS_NAMES, list(out)))

    def set_timing(self, on: bool):
        _check(lib().tawpipe_set_timing(1 if on else 0))

    def trace(self) -> dict:
        """Trace-Event JSON of the last timed step (tawpipe_trace_json), parsed; {} before any timed step."""
        n = lib().tawpipe_trace_json(None, 0)
        if n < 0:
            _check(int(n))
        if n == 0:
            return {}
        buf = ctypes.create_string_buffer(int(n) + 1)
        lib().tawpipe_trace_json(buf, n + 1)
        import json
        return json.loads(buf.value.decode())

    def set_link_emulation(self, inter_gbps: float, latency_us: float = 0.0, node_size: int = 0):
        """Pace transfers that cross emulated node boundaries (tawpipe_set_link_emulation); 0 GB/s disables."""
        _check(lib().tawpipe_set_link_emulation(float(inter_gbps), float(latency_us), int(node_size)))

    def close(self):
        lib().tawpipe_finalize()


def plan(n_devices: int, group_size: int, dims: ModelDims, n_micro: int, rank: int):
    """Host-only dry run (tawpipe_plan): (ledger list, shard elements) of `rank`; raises on invalid config."""
    led = (ctypes.c_uint64 * LEDGER_N)()
    n = ctypes.c_int64(0)
    cd = dims.to_c()
    _check(lib().tawpipe_plan(n_devices, group_size, dims.n_layers, ctypes.byref(cd), n_micro, rank, led,
                              ctypes.byref(n)))
    return [int(x) for x in led], int(n.value)


# ---------------------------------------------------------------------------------------------- kernel-level
def gemm(dtype, M, N, K, A, a_ld, a_kmajor, B, b_ld, b_kmajor, C, c_ld, c_f32=False, accumulate=False, R=None,
         stream=None):
    """Device-pointer GEMM C (+)= A·Bᵀ (see include/tawpipe.h)."""
    _check(lib().tawpipe_gemm(dtype, M, N, K, A, a_ld, int(a_kmajor), B, b_ld, int(b_kmajor), C, c_ld, int(c_f32),
                              int(accumulate), R, stream))


def attention_fwd(dtype, B, S, nh, dh, qkv, o, lse, stream=None):
    _check(lib().tawpipe_attention_fwd(dtype, B, S, nh, dh, qkv, o, lse, stream))


def attention_bwd(dtype, B, S, nh, dh, qkv, o, lse, do, dqkv, scratch, dq_acc, stream=None):
    """scratch: 2·B·n_h·S fp32 (δ and the log2-domain LSE)."""
    _check(lib().tawpipe_attention_bwd(dtype, B, S, nh, dh, qkv, o, lse, do, dqkv, scratch, dq_acc, stream))


def attention_bwd_rope(dtype, B, S, nh, dh, theta, qkv, o, lse, do, dqkv, scratch, dq_acc, stream=None):
    _check(lib().tawpipe_attention_bwd_rope(dtype, B, S, nh, dh, theta, qkv, o, lse, do, dqkv, scratch, dq_acc,
                                            stream))


def gemm_rope(M, N, K, x, w, qkv, S, dh, theta, rope_cols, stream=None):
    _check(lib().tawpipe_gemm_rope(M, N, K, x, w, qkv, S, dh, theta, rope_cols, stream))


def gemm_swiglu(M, I, K, x, w_gu, gu, y, stream=None):
    _check(lib().tawpipe_gemm_swiglu(M, I, K, x, w_gu, gu, y, stream))


def gemm_swiglu_bwd(M, I, K, dh, w_down, gu, dgu, stream=None):
    _check(lib().tawpipe_gemm_swiglu_bwd(M, I, K, dh, w_down, gu, dgu, stream))


def rmsnorm_fwd(dtype, rows, H, x, gamma, eps, y, rstd, stream=None):
    _check(lib().tawpipe_rmsnorm_fwd(dtype, rows, H, x, gamma, eps, y, rstd, stream))


def rmsnorm_bwd(dtype, rows, H, dy, x, gamma, rstd, res, dx, dgamma_acc, stream=None):
    _check(lib().tawpipe_rmsnorm_bwd(dtype, rows, H, dy, x, gamma, rstd, res, dx, dgamma_acc, stream))


def rope(dtype, B, S, nh, dh, theta, qkv, inverse, stream=None):
    _check(lib().tawpipe_rope(dtype, B, S, nh, dh, theta, qkv, int(inverse), stream))


def swiglu_fwd(dtype, rows, I, gu, y, stream=None):
    _check(lib().tawpipe_swiglu_fwd(dtype, rows, I, gu, y, stream))


def swiglu_bwd(dtype, rows, I, dy, gu, dgu, stream=None):
    _check(lib().tawpipe_swiglu_bwd(dtype, rows, I, dy, gu, dgu, stream))


def cross_entropy(dtype, rows, V, logits, targets, inv_denom, loss_rows, stream=None):
    _check(lib().tawpipe_cross_entropy(dtype, rows, V, logits, targets, inv_denom, loss_rows, stream))


def embed_fwd(dtype, B, S, tokens, tok_stride, E, H, h, stream=None):
    _check(lib().tawpipe_embed_fwd(dtype, B, S, tokens, tok_stride, E, H, h, stream))


def embed_bwd(dtype, B, S, tokens, tok_stride, dh, H, V, dE, stream=None):
    _check(lib().tawpipe_embed_bwd(dtype, B, S, tokens, tok_stride, dh, H, V, dE, stream))


def group_partial(wire_dtype, srcs, n, out, stream=None):
    """srcs: device pointers of n fp32 elements, summed in list order into out (wire dtype) (tawpipe_group_partial)."""
    ptrs = (ctypes.c_void_p * len(srcs))(*srcs)
    _check(lib().tawpipe_group_partial(wire_dtype, len(srcs), ptrs, n, out, stream))


def adamw(wire_dtype, groups, master, m, v, wire, n, unit_off=0, no_decay=None, lr=1e-3, beta1=0.9, beta2=0.95,
          eps=1e-8, wd=0.1, step=1, stream=None):
    """groups: list of groups, each a list of (device pointer, is_f32) sources summed in member order, the groups in
    list order (tawpipe_adamw)."""
    sizes = (ctypes.c_int * len(groups))(*[len(gr) for gr in groups])
    flat = [src for gr in groups for src in gr]
    ptrs = (ctypes.c_void_p * len(flat))(*[p for p, _ in flat])
    f32 = (ctypes.c_int * len(flat))(*[int(bool(f)) for _, f in flat])
    nd = None if no_decay is None else (ctypes.c_int64 * 4)(*no_decay)
    hyper = (ctypes.c_float * 5)(lr, beta1, beta2, eps, wd)
    _check(lib().tawpipe_adamw(wire_dtype, len(groups), sizes, ptrs, f32, master, m, v, wire, n, unit_off, nd, hyper,
                               step, stream))
