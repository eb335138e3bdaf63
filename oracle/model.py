"""Plain fp64 LLaMA-style decoder forward / backward and AdamW (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Every function follows SURVEY.md §8(c) "Algorithm, step by step" and the
backward-formula table there, which restate the paper's model: a LLaMA-2-derived
decoder (§4.1) trained with AdamW on "colocated optimizer states"
(§3.3).  Readings of silent points are SURVEY.md §8(c) R1-R21 and
are listed in DESIGN.md §Readings.  No blocking, fusion or reordering: each op
is its textbook definition, one sequence at a time.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


# ----------------------------------------------------------------------------
# configuration
# ----------------------------------------------------------------------------
@dataclass
class ModelConfig:
    n_layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    seq: int
    micro_bs: int = 1
    rms_eps: float = 1e-5          # R10
    rope_theta: float = 10000.0    # R10
    # AdamW, PyTorch semantics (R1)
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    weight_decay: float = 0.1

    @property
    def head_dim(self) -> int:
        assert self.hidden % self.heads == 0
        return self.hidden // self.heads


# Parameter names of one decoder layer in canonical order:
# [attn_norm H | Wq H·H | Wk H·H | Wv H·H | Wo H·H | mlp_norm H | Wgate I·H | Wup I·H | Wdown H·I]
LAYER_KEYS = ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "w_gate", "w_up", "w_down")
NO_DECAY = ("attn_norm", "mlp_norm", "final_norm")   # R1: no weight decay on RMSNorm gains


def layer_shapes(cfg: ModelConfig):
    H, I = cfg.hidden, cfg.ffn
    return {"attn_norm": (H,), "wq": (H, H), "wk": (H, H), "wv": (H, H), "wo": (H, H),
            "mlp_norm": (H,), "w_gate": (I, H), "w_up": (I, H), "w_down": (H, I)}


def phi(cfg: ModelConfig) -> int:
    """Exact parameter count of one decoder layer: 4H² + 3HI + 2H (SURVEY.md §0 notation)."""
    H, I = cfg.hidden, cfg.ffn
    return 4 * H * H + 3 * H * I + 2 * H


def to_f64(params: dict) -> dict:
    return {"embed": params["embed"].astype(np.float64),
            "layers": [{k: v.astype(np.float64) for k, v in lay.items()} for lay in params["layers"]],
            "final_norm": params["final_norm"].astype(np.float64),
            "head": params["head"].astype(np.float64)}


def zeros_like_params(p: dict) -> dict:
    return {"embed": np.zeros_like(p["embed"]),
            "layers": [{k: np.zeros_like(v) for k, v in lay.items()} for lay in p["layers"]],
            "final_norm": np.zeros_like(p["final_norm"]), "head": np.zeros_like(p["head"])}


# ----------------------------------------------------------------------------
# per-op forward / backward (SURVEY.md §8(c) backward-formula table)
# ----------------------------------------------------------------------------
def rmsnorm_fwd(x, g, eps):
    """y = x · r ⊙ γ with r = (mean_H(x²) + ε)^(-1/2), row-wise."""
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * g, r


def rmsnorm_bwd(dy, x, g, r):
    """dγ = Σ_rows dy⊙x·r ;  with gg = dy⊙γ:  dx = r·gg − x·r³·mean_H(gg⊙x)."""
    dg = np.sum(dy * x * r, axis=0)
    gg = dy * g
    dx = r * gg - x * (r ** 3) * np.mean(gg * x, axis=-1, keepdims=True)
    return dx, dg


def rope_tables(seq, head_dim, theta):
    """cos/sin [S, d_h/2] of p·θ_i, θ_i = base^(−2i/d_h) (rotate-half convention, R10/R13)."""
    half = head_dim // 2
    i = np.arange(half, dtype=np.float64)
    inv = theta ** (-2.0 * i / head_dim)
    ang = np.arange(seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope_fwd(x, cos, sin):
    """x [S, n_h, d_h]:  x'_i = x_i cos − x_{i+d/2} sin ;  x'_{i+d/2} = x_{i+d/2} cos + x_i sin."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rope_bwd(dy, cos, sin):
    """Rotation by −pθ_i:  dx_i = dy_i cos + dy_{i+d/2} sin ;  dx_{i+d/2} = dy_{i+d/2} cos − dy_i sin."""
    half = dy.shape[-1] // 2
    d1, d2 = dy[..., :half], dy[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([d1 * c + d2 * s, d2 * c - d1 * s], axis=-1)


def attention_fwd(q, k, v):
    """Causal softmax attention per head; q,k,v [S, n_h, d_h] -> o [S, n_h, d_h], P [n_h, S, S].

    S = c·q k^T with c = 1/sqrt(d_h), −∞ where key > query; P = row-softmax
    (row max subtracted); o = P v.
    """
    S_, nh, dh = q.shape
    c = 1.0 / np.sqrt(dh)
    mask = np.triu(np.ones((S_, S_), dtype=bool), k=1)
    o = np.empty_like(q)
    P = np.empty((nh, S_, S_))
    for h in range(nh):
        s = c * (q[:, h, :] @ k[:, h, :].T)
        s[mask] = -np.inf
        s = s - s.max(axis=1, keepdims=True)
        e = np.exp(s)
        P[h] = e / e.sum(axis=1, keepdims=True)
        o[:, h, :] = P[h] @ v[:, h, :]
    return o, P


def attention_bwd(do, q, k, v, o, P):
    """dv = Pᵀ do; dP = do vᵀ; δ = rowsum(do⊙o); dS = P⊙(dP − δ); dq = c dS k; dk = c dSᵀ q."""
    S_, nh, dh = q.shape
    c = 1.0 / np.sqrt(dh)
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    for h in range(nh):
        dv[:, h, :] = P[h].T @ do[:, h, :]
        dP = do[:, h, :] @ v[:, h, :].T
        delta = np.sum(do[:, h, :] * o[:, h, :], axis=1, keepdims=True)
        dS = P[h] * (dP - delta)
        dq[:, h, :] = c * (dS @ k[:, h, :])
        dk[:, h, :] = c * (dS.T @ q[:, h, :])
    return dq, dk, dv


def attention_row(i, q_i, k, v, do_i):
    """One query row of attention_fwd / attention_bwd for one head, for spot checks at sizes where the S×S
    matrices do not fit: keys 0..i only (causal), the same definitions row by row.  q_i, do_i [d_h];
    k, v [S, d_h].  Returns (o_i, lse_i, dq_i) with lse_i = log Σ_j exp(c·q_i·k_j)."""
    dh = q_i.shape[0]
    c = 1.0 / np.sqrt(dh)
    s = c * (k[: i + 1] @ q_i)
    mx = s.max()
    e = np.exp(s - mx)
    lse = mx + np.log(e.sum())
    p = e / e.sum()
    o_i = p @ v[: i + 1]
    dP = v[: i + 1] @ do_i
    delta = float(do_i @ o_i)
    dS = p * (dP - delta)
    dq_i = c * (dS @ k[: i + 1])
    return o_i, lse, dq_i


def attention_fwd_rows(i0, i1, q, k, v):
    """Query rows i0..i1−1 of attention_fwd for one head, with their LSE: the same definition evaluated for a
    subset of rows (each row is independent), for spot checks at sizes where the S×S matrices do not fit.
    q, k, v [S, d_h].  Returns (o [i1−i0, d_h], lse [i1−i0]) with lse_i = log Σ_{j ≤ i} exp(c·q_i·k_j)."""
    dh = q.shape[1]
    c = 1.0 / np.sqrt(dh)
    s = c * (q[i0:i1] @ k[:i1].T)                              # [rows, i1]
    s[np.arange(i1)[None, :] > np.arange(i0, i1)[:, None]] = -np.inf   # causal: key j > query i masked
    mx = s.max(axis=1, keepdims=True)
    e = np.exp(s - mx)
    se = e.sum(axis=1, keepdims=True)
    return (e / se) @ v[:i1], (mx + np.log(se))[:, 0]


def attention_key_row(j, k_j, v_j, q, do, o, lse):
    """Key row j of attention_bwd for one head: only query rows i ≥ j see key j (causal).
    P_ij = exp(c·q_i·k_j − lse_i); dV_j = Σ_i P_ij do_i; dP_ij = do_i·v_j; δ_i = do_i·o_i; dS_ij = P_ij (dP_ij − δ_i);
    dK_j = c Σ_i dS_ij q_i.  q, do, o [S, d_h] and lse [S] cover rows 0..S−1 (rows < j are not read)."""
    dh = q.shape[1]
    c = 1.0 / np.sqrt(dh)
    qi, doi, oi = q[j:], do[j:], o[j:]
    p = np.exp(c * (qi @ k_j) - lse[j:])
    dv_j = p @ doi
    dP = doi @ v_j
    delta = np.sum(doi * oi, axis=1)
    dS = p * (dP - delta)
    dk_j = c * (dS @ qi)
    return dk_j, dv_j


def sigmoid(u):
    return 1.0 / (1.0 + np.exp(-u))


def swiglu_fwd(u, w):
    """y = SiLU(u) ⊙ w, SiLU(u) = u·σ(u)."""
    return u * sigmoid(u) * w


def swiglu_bwd(dy, u, w):
    """du = dy⊙w⊙σ(u)(1 + u(1−σ(u))) ;  dw = dy⊙SiLU(u)."""
    sg = sigmoid(u)
    du = dy * w * sg * (1.0 + u * (1.0 - sg))
    dw = dy * u * sg
    return du, dw


def cross_entropy_fwd_bwd(z, targets, denom):
    """ℓ = Σ_p [LSE(z_p) − z_p[t_p]];  dz_p = (softmax(z_p) − onehot(t_p)) / denom."""
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    se = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(se))[:, 0]
    rows = np.arange(z.shape[0])
    loss = float(np.sum(lse - z[rows, targets]))
    dz = e / se
    dz[rows, targets] -= 1.0
    return loss, dz / denom


# ----------------------------------------------------------------------------
# one decoder layer on one sequence (§8(a) a5 / a7)
# ----------------------------------------------------------------------------
def layer_fwd(h, W, cfg: ModelConfig, cos, sin):
    S_, H = h.shape
    nh, dh = cfg.heads, cfg.head_dim
    a, r1 = rmsnorm_fwd(h, W["attn_norm"], cfg.rms_eps)
    q = (a @ W["wq"].T).reshape(S_, nh, dh)
    k = (a @ W["wk"].T).reshape(S_, nh, dh)
    v = (a @ W["wv"].T).reshape(S_, nh, dh)
    qr, kr = rope_fwd(q, cos, sin), rope_fwd(k, cos, sin)
    o, P = attention_fwd(qr, kr, v)
    o2 = o.reshape(S_, H)
    h1 = h + o2 @ W["wo"].T
    b, r2 = rmsnorm_fwd(h1, W["mlp_norm"], cfg.rms_eps)
    u = b @ W["w_gate"].T
    w = b @ W["w_up"].T
    y = swiglu_fwd(u, w)
    h2 = h1 + y @ W["w_down"].T
    cache = dict(h=h, a=a, r1=r1, qr=qr, kr=kr, v=v, o=o, P=P, o2=o2, h1=h1, b=b, r2=r2, u=u, w=w, y=y)
    return h2, cache


def layer_bwd(dh2, W, c, cfg: ModelConfig, cos, sin):
    """Returns dh and this sequence's gradient dict for the layer."""
    S_, H = dh2.shape
    nh, dh = cfg.heads, cfg.head_dim
    g = {}
    # h2 = h1 + y·Wdownᵀ
    g["w_down"] = dh2.T @ c["y"]
    dy = dh2 @ W["w_down"]
    du, dw = swiglu_bwd(dy, c["u"], c["w"])
    g["w_gate"] = du.T @ c["b"]
    g["w_up"] = dw.T @ c["b"]
    db = du @ W["w_gate"] + dw @ W["w_up"]
    dh1_n, g["mlp_norm"] = rmsnorm_bwd(db, c["h1"], W["mlp_norm"], c["r2"])
    dh1 = dh2 + dh1_n
    # h1 = h + o·Woᵀ
    g["wo"] = dh1.T @ c["o2"]
    do = (dh1 @ W["wo"]).reshape(S_, nh, dh)
    dqr, dkr, dv = attention_bwd(do, c["qr"], c["kr"], c["v"], c["o"], c["P"])
    dq = rope_bwd(dqr, cos, sin).reshape(S_, H)
    dk = rope_bwd(dkr, cos, sin).reshape(S_, H)
    dv = dv.reshape(S_, H)
    g["wq"] = dq.T @ c["a"]
    g["wk"] = dk.T @ c["a"]
    g["wv"] = dv.T @ c["a"]
    da = dq @ W["wq"] + dk @ W["wk"] + dv @ W["wv"]
    dh_n, g["attn_norm"] = rmsnorm_bwd(da, c["h"], W["attn_norm"], c["r1"])
    return dh1 + dh_n, g


def head_fwd_bwd(h, final_norm, head, targets, denom, cfg: ModelConfig):
    """f = RMSNorm(h; γ_f); z = f·W_headᵀ; CE."""
    f, r = rmsnorm_fwd(h, final_norm, cfg.rms_eps)
    z = f @ head.T
    loss, dz = cross_entropy_fwd_bwd(z, targets, denom)
    d_head = dz.T @ f
    df = dz @ head
    dh, d_fn = rmsnorm_bwd(df, h, final_norm, r)
    return loss, dh, d_fn, d_head


# ----------------------------------------------------------------------------
# whole model: loss and gradients of the global mean (R2), one sequence at a time
# ----------------------------------------------------------------------------
def sequence_loss_and_grads(P64, seq_tokens, cfg: ModelConfig, denom, grads, cos, sin):
    """Adds this sequence's gradient contribution into ``grads``; returns its loss sum ℓ_seq."""
    x, t = seq_tokens[:-1], seq_tokens[1:]
    h = P64["embed"][x]                       # step 1: h = E[x]
    caches = []
    for W in P64["layers"]:                   # step 2
        h, cch = layer_fwd(h, W, cfg, cos, sin)
        caches.append(cch)
    loss, dh, d_fn, d_head = head_fwd_bwd(h, P64["final_norm"], P64["head"], t, denom, cfg)
    grads["final_norm"] += d_fn
    grads["head"] += d_head
    for li in range(len(P64["layers"]) - 1, -1, -1):
        dh, g = layer_bwd(dh, P64["layers"][li], caches[li], cfg, cos, sin)
        for k_, v_ in g.items():
            grads["layers"][li][k_] += v_
    np.add.at(grads["embed"], x, dh)          # dE[x_p] += dh0[p], sequential
    return loss


def loss_and_grads(params, tokens, cfg: ModelConfig):
    """Global mean loss over all N·B·S predicted tokens (R2) and its exact gradient.

    tokens int [N][B][S+1] (R3).  Returns (loss, grads) in float64.
    """
    P64 = to_f64(params) if params["embed"].dtype != np.float64 else params
    N, B, S1 = tokens.shape
    assert S1 == cfg.seq + 1
    denom = float(N * B * cfg.seq)
    cos, sin = rope_tables(cfg.seq, cfg.head_dim, cfg.rope_theta)
    grads = zeros_like_params(P64)
    total = 0.0
    for n in range(N):
        for b in range(B):
            total += sequence_loss_and_grads(P64, tokens[n, b], cfg, denom, grads, cos, sin)
    return total / denom, grads


# ----------------------------------------------------------------------------
# AdamW (PyTorch torch.optim.AdamW semantics, R1)
# ----------------------------------------------------------------------------
def adamw_update(theta, g, m, v, t, cfg: ModelConfig, decay: bool):
    """One AdamW step on arrays (returns new θ, m, v).

    θ ← θ(1 − lr·wd) if decayed; m ← β1 m + (1−β1) g; v ← β2 v + (1−β2) g²;
    θ ← θ − lr·(m/(1−β1ᵗ)) / (sqrt(v/(1−β2ᵗ)) + ε).
    """
    lr, b1, b2, eps, wd = cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps, cfg.weight_decay
    if decay:
        theta = theta * (1.0 - lr * wd)
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mhat = m / (1.0 - b1 ** t)
    vhat = v / (1.0 - b2 ** t)
    theta = theta - lr * mhat / (np.sqrt(vhat) + eps)
    return theta, m, v


@dataclass
class TrainState:
    params: dict                      # float64
    m: dict
    v: dict
    t: int = 0
    losses: list = field(default_factory=list)


def init_state(params) -> TrainState:
    p = to_f64(params)
    return TrainState(params=p, m=zeros_like_params(p), v=zeros_like_params(p))


def apply_adamw(state: TrainState, grads, cfg: ModelConfig):
    state.t += 1
    t = state.t
    for name in ("embed", "head", "final_norm"):
        state.params[name], state.m[name], state.v[name] = adamw_update(
            state.params[name], grads[name], state.m[name], state.v[name], t, cfg,
            decay=name not in NO_DECAY)
    for li, lay in enumerate(state.params["layers"]):
        for k_ in LAYER_KEYS:
            lay[k_], state.m["layers"][li][k_], state.v["layers"][li][k_] = adamw_update(
                lay[k_], grads["layers"][li][k_], state.m["layers"][li][k_],
                state.v["layers"][li][k_], t, cfg, decay=k_ not in NO_DECAY)


def train_step(state: TrainState, tokens, cfg: ModelConfig):
    """One synchronous iteration: global-mean loss, exact gradients, one AdamW update."""
    loss, grads = loss_and_grads(state.params, tokens, cfg)
    apply_adamw(state, grads, cfg)
    state.losses.append(loss)
    return loss, grads
