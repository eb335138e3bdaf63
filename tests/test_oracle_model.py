"""Pins of the fp64 oracle model against things other than itself (SURVEY.md §8(c) pin table).

- finite differences on a micro-config (brute force on tiny inputs);
- an independent torch-fp64 autograd model + torch.optim.AdamW (library routines);
- closed forms / invariants of each op.
"""
import math

import numpy as np
import pytest

import synth
from oracle import model as om

MICRO = dict(n_layers=2, hidden=16, heads=2, ffn=48, vocab=32, seq=8, micro_bs=1)


def micro_cfg(**kw):
    d = dict(MICRO)
    d.update(kw)
    return om.ModelConfig(**d)


def micro_params(cfg, seed=1234, gains=True):
    p = synth.init_params(cfg.n_layers, cfg.hidden, cfg.ffn, cfg.vocab, seed=seed)
    # larger weights than N(0,0.02) so that every term of the backward matters
    p = {"embed": p["embed"] * 25, "head": p["head"] * 25, "final_norm": p["final_norm"],
         "layers": [{k: (v * 15 if v.ndim == 2 else v) for k, v in lay.items()} for lay in p["layers"]]}
    return synth.perturb_gains(p, scale=0.3) if gains else p


# --------------------------------------------------------------------------- finite differences
def test_finite_differences_all_tensors():
    cfg = micro_cfg()
    params = om.to_f64(micro_params(cfg))
    toks = synth.tokens(2, 1, cfg.seq, cfg.vocab, step=3)
    loss, grads = om.loss_and_grads(params, toks, cfg)
    rng = np.random.default_rng(0)
    h = 1e-5

    def loss_at(path, idx, delta):
        obj = params
        for p_ in path[:-1]:
            obj = obj[p_]
        arr = obj[path[-1]]
        old = arr[idx]
        arr[idx] = old + delta
        val, _ = om.loss_and_grads(params, toks, cfg)
        arr[idx] = old
        return val

    paths = [("embed",), ("head",), ("final_norm",)]
    for li in range(cfg.n_layers):
        paths += [("layers", li, k) for k in om.LAYER_KEYS]
    checked = 0
    for path in paths:
        g = grads
        arr = params
        for p_ in path:
            g = g[p_]
            arr = arr[p_]
        gmax = np.abs(g).max()
        n = 12 if path[0] != "embed" else 8
        flat_idx = rng.choice(arr.size, size=min(n, arr.size), replace=False)
        if path[0] == "embed":    # rows of tokens that actually occur
            rows = np.unique(toks[:, :, :-1])
            flat_idx = [int(rows[i % len(rows)]) * cfg.hidden + int(c)
                        for i, c in enumerate(rng.integers(0, cfg.hidden, n))]
        for fi in flat_idx:
            idx = np.unravel_index(int(fi), arr.shape)
            fd = (loss_at(path, idx, h) - loss_at(path, idx, -h)) / (2 * h)
            an = g[idx]
            assert abs(fd - an) <= 1e-6 * max(abs(an), 1e-4 * gmax) + 2e-10, (path, idx, fd, an)
            checked += 1
    assert checked >= 200


# --------------------------------------------------------------------------- torch fp64 re-derivation
def torch_reference_step(params, toks, cfg, n_steps=1):
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    t = lambda a: torch.tensor(np.asarray(a, np.float64), requires_grad=True)
    P = {"embed": t(params["embed"]), "head": t(params["head"]), "final_norm": t(params["final_norm"]),
         "layers": [{k: t(v) for k, v in lay.items()} for lay in params["layers"]]}
    decay = [P["embed"], P["head"]] + [lay[k] for lay in P["layers"] for k in om.LAYER_KEYS
                                       if k not in ("attn_norm", "mlp_norm")]
    nodecay = [P["final_norm"]] + [lay[k] for lay in P["layers"] for k in ("attn_norm", "mlp_norm")]
    opt = torch.optim.AdamW([{"params": decay, "weight_decay": cfg.weight_decay},
                             {"params": nodecay, "weight_decay": 0.0}],
                            lr=cfg.lr, betas=(cfg.beta1, cfg.beta2), eps=cfg.adam_eps, foreach=False)
    nh, dh, S = cfg.heads, cfg.head_dim, cfg.seq
    # RoPE written in the complex form (x_i + i x_{i+d/2}) · e^{i p θ_i}: a different formulation
    inv = cfg.rope_theta ** (-torch.arange(dh // 2, dtype=torch.float64) * 2 / dh)
    rot = torch.polar(torch.ones(S, dh // 2, dtype=torch.float64),
                      torch.arange(S, dtype=torch.float64)[:, None] * inv[None, :])

    def rope(x):  # x [S, nh, dh]
        c = torch.complex(x[..., :dh // 2], x[..., dh // 2:]) * rot[:, None, :]
        return torch.cat([c.real, c.imag], dim=-1)

    losses = []
    for _ in range(n_steps):
        opt.zero_grad()
        N, B, _ = toks.shape
        total = 0.0
        for n in range(N):
            for b in range(B):
                x = torch.tensor(toks[n, b, :-1].astype(np.int64))
                y = torch.tensor(toks[n, b, 1:].astype(np.int64))
                h = P["embed"][x]
                for W in P["layers"]:
                    a = F.rms_norm(h, (cfg.hidden,), W["attn_norm"], eps=cfg.rms_eps)
                    q = rope((a @ W["wq"].T).view(S, nh, dh)).transpose(0, 1)
                    k = rope((a @ W["wk"].T).view(S, nh, dh)).transpose(0, 1)
                    v = (a @ W["wv"].T).view(S, nh, dh).transpose(0, 1)
                    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                    h = h + o.transpose(0, 1).reshape(S, cfg.hidden) @ W["wo"].T
                    bb = F.rms_norm(h, (cfg.hidden,), W["mlp_norm"], eps=cfg.rms_eps)
                    h = h + (F.silu(bb @ W["w_gate"].T) * (bb @ W["w_up"].T)) @ W["w_down"].T
                f = F.rms_norm(h, (cfg.hidden,), P["final_norm"], eps=cfg.rms_eps)
                total = total + F.cross_entropy(f @ P["head"].T, y, reduction="sum")
        loss = total / (N * B * S)
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    out = {"embed": P["embed"].detach().numpy(), "head": P["head"].detach().numpy(),
           "final_norm": P["final_norm"].detach().numpy(),
           "layers": [{k: v.detach().numpy() for k, v in lay.items()} for lay in P["layers"]]}
    return losses, out


def flat(p):
    parts = [p["embed"].ravel(), p["head"].ravel(), p["final_norm"].ravel()]
    for lay in p["layers"]:
        parts += [lay[k].ravel() for k in om.LAYER_KEYS]
    return np.concatenate(parts)


def test_matches_torch_fp64_autograd_and_adamw_three_steps():
    cfg = micro_cfg(micro_bs=2)
    params = micro_params(cfg)
    toks = synth.tokens(2, 2, cfg.seq, cfg.vocab, step=5)
    st = om.init_state(params)
    losses = [om.train_step(st, toks, cfg)[0] for _ in range(3)]
    tl, tp = torch_reference_step(params, toks, cfg, n_steps=3)
    np.testing.assert_allclose(losses, tl, rtol=1e-12)
    a, b = flat(st.params), flat(tp)
    assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= 1e-12


# --------------------------------------------------------------------------- closed forms / invariants
def test_zero_head_gives_ln_V_and_onehot_gradient():
    cfg = micro_cfg()
    params = om.to_f64(micro_params(cfg))
    params["head"][:] = 0.0
    toks = synth.tokens(2, 1, cfg.seq, cfg.vocab, step=1)
    loss, grads = om.loss_and_grads(params, toks, cfg)
    assert abs(loss - math.log(cfg.vocab)) <= 1e-14 * math.log(cfg.vocab)
    # dlogits = (1/V - onehot)/(N·B·S); nothing flows back through W_head = 0
    assert np.all(grads["embed"] == 0) and np.all(grads["final_norm"] == 0)
    for lay in grads["layers"]:
        assert all(np.all(v == 0) for v in lay.values())
    # d_head = Σ_p dz_pᵀ f_p: recompute f from the forward to check the closed form
    denom = 2 * cfg.seq
    dh_expect = np.zeros_like(params["head"])
    cos, sin = om.rope_tables(cfg.seq, cfg.head_dim, cfg.rope_theta)
    for n in range(2):
        x, t = toks[n, 0, :-1], toks[n, 0, 1:]
        h = params["embed"][x]
        for W in params["layers"]:
            h, _ = om.layer_fwd(h, W, cfg, cos, sin)
        f, _ = om.rmsnorm_fwd(h, params["final_norm"], cfg.rms_eps)
        dz = np.full((cfg.seq, cfg.vocab), 1.0 / cfg.vocab)
        dz[np.arange(cfg.seq), t] -= 1.0
        dh_expect += (dz / denom).T @ f
    np.testing.assert_allclose(grads["head"], dh_expect, rtol=1e-12, atol=1e-15)


def test_rmsnorm_invariants():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((5, 24)) * 3
    y, r = om.rmsnorm_fwd(x, np.ones(24), 1e-5)
    np.testing.assert_allclose(np.sqrt(np.mean(y * y, axis=1)), 1.0, rtol=1e-5)
    y0, _ = om.rmsnorm_fwd(x, np.ones(24), 0.0)
    y1, _ = om.rmsnorm_fwd(7.5 * x, np.ones(24), 0.0)
    np.testing.assert_allclose(y0, y1, rtol=1e-13)
    g = rng.uniform(0.5, 1.5, 24)
    dy = rng.standard_normal((5, 24))
    _, r0 = om.rmsnorm_fwd(x, g, 0.0)
    dx, _ = om.rmsnorm_bwd(dy, x, g, r0)
    np.testing.assert_allclose(np.sum(x * dx, axis=1), 0.0, atol=1e-12)
    eps = 0.3
    _, re = om.rmsnorm_fwd(x, g, eps)
    dx, _ = om.rmsnorm_bwd(dy, x, g, re)
    ms = np.mean(x * x, axis=1)
    expect = re[:, 0] * np.sum(dy * g * x, axis=1) * eps / (ms + eps)
    np.testing.assert_allclose(np.sum(x * dx, axis=1), expect, rtol=1e-12)


def test_rope_invariants():
    rng = np.random.default_rng(2)
    S, nh, dh = 9, 3, 8
    cos, sin = om.rope_tables(S, dh, 10000.0)
    q = rng.standard_normal((S, nh, dh))
    k = rng.standard_normal((S, nh, dh))
    qr, kr = om.rope_fwd(q, cos, sin), om.rope_fwd(k, cos, sin)
    np.testing.assert_allclose(np.linalg.norm(qr, axis=-1), np.linalg.norm(q, axis=-1), rtol=1e-13)
    np.testing.assert_allclose(qr[0], q[0], rtol=0, atol=0)
    # <RoPE_p(q), RoPE_r(k)> depends only on p − r: same vector at every position
    qq = np.broadcast_to(q[0], (S, nh, dh)).copy()
    kk = np.broadcast_to(k[0], (S, nh, dh)).copy()
    qqr, kkr = om.rope_fwd(qq, cos, sin), om.rope_fwd(kk, cos, sin)
    d1 = np.sum(qqr[5] * kkr[2], axis=-1)
    d2 = np.sum(qqr[7] * kkr[4], axis=-1)
    np.testing.assert_allclose(d1, d2, rtol=1e-12)
    # backward is the inverse (transpose) rotation
    np.testing.assert_allclose(om.rope_bwd(qr, cos, sin), q, rtol=1e-12, atol=1e-14)
    # position p, i = 0 rotates by angle p exactly (θ_0 = 1)
    e = np.zeros((S, 1, dh))
    e[:, 0, 0] = 1.0
    er = om.rope_fwd(e, cos, sin)
    np.testing.assert_allclose(er[:, 0, 0], np.cos(np.arange(S)), rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(er[:, 0, dh // 2], np.sin(np.arange(S)), rtol=1e-14, atol=1e-15)


def test_attention_closed_forms():
    rng = np.random.default_rng(3)
    S, nh, dh = 7, 2, 4
    q = rng.standard_normal((S, nh, dh))
    k = rng.standard_normal((S, nh, dh))
    v = rng.standard_normal((S, nh, dh))
    o, P = om.attention_fwd(q, k, v)
    np.testing.assert_allclose(o[0], v[0], rtol=1e-14)
    o0, _ = om.attention_fwd(np.zeros_like(q), k, v)
    prefix = np.cumsum(v, axis=0) / np.arange(1, S + 1)[:, None, None]
    np.testing.assert_allclose(o0, prefix, rtol=1e-13)
    o1, _ = om.attention_fwd(q[:1], k[:1], v[:1])
    np.testing.assert_allclose(o1, v[:1], rtol=1e-14)
    assert np.all(np.triu(P[0], 1) == 0)
    np.testing.assert_allclose(P.sum(-1), 1.0, rtol=1e-14)


def test_attention_row_form_equals_matrix_form_and_closed_forms():
    """oracle.attention_row (full-size spot checks) agrees with the pinned matrix form row by row, and on its own
    reproduces the closed forms: row 0 attends only to key 0 (o_0 = v_0, dq_0 = 0), a zero query gives the prefix
    mean, and lse of a zero query is log(i + 1)."""
    rng = np.random.default_rng(4)
    S, nh, dh = 9, 2, 8
    q, k, v, do = (rng.standard_normal((S, nh, dh)) for _ in range(4))
    o, P = om.attention_fwd(q, k, v)
    dq, _, _ = om.attention_bwd(do, q, k, v, o, P)
    for h in range(nh):
        for i in range(S):
            oi, lse, dqi = om.attention_row(i, q[i, h], k[:, h], v[:, h], do[i, h])
            np.testing.assert_allclose(oi, o[i, h], rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(dqi, dq[i, h], rtol=1e-11, atol=1e-13)
            s_ = (k[: i + 1, h] @ q[i, h]) / np.sqrt(dh)
            assert abs(lse - np.log(np.sum(np.exp(s_)))) < 1e-12
    o0, lse0, dq0 = om.attention_row(0, q[0, 0], k[:, 0], v[:, 0], do[0, 0])
    np.testing.assert_allclose(o0, v[0, 0], rtol=1e-14)
    np.testing.assert_allclose(dq0, 0.0, atol=1e-14)
    oz, lz, _ = om.attention_row(5, np.zeros(dh), k[:, 0], v[:, 0], do[5, 0])
    np.testing.assert_allclose(oz, v[:6, 0].mean(0), rtol=1e-13)
    assert abs(lz - np.log(6)) < 1e-14


def test_swiglu_closed_forms():
    u = np.linspace(-4, 4, 33)
    w = np.linspace(1, 2, 33)
    assert np.all(om.swiglu_fwd(np.zeros(5), np.ones(5)) == 0)
    du, dw = om.swiglu_bwd(np.ones_like(u), u, w)
    h = 1e-5
    fd = ((u + h) / (1 + np.exp(-(u + h))) - (u - h) / (1 + np.exp(-(u - h)))) / (2 * h)
    np.testing.assert_allclose(du, fd * w, rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(dw, u / (1 + np.exp(-u)), rtol=1e-14)


def test_adamw_step1_closed_form_and_step2_by_hand():
    cfg = micro_cfg()
    theta = np.array([0.5, -0.25, 1.0, 0.0])
    g = np.array([0.1, -0.02, 0.0, 3.0])
    th1, m1, v1 = om.adamw_update(theta, g, np.zeros(4), np.zeros(4), 1, cfg, decay=True)
    expect = theta * (1 - cfg.lr * cfg.weight_decay) - cfg.lr * g / (np.abs(g) + cfg.adam_eps)
    np.testing.assert_allclose(th1, expect, rtol=1e-15, atol=1e-18)
    g2 = np.array([-0.05, 0.04, 1.0, 1.0])
    th2, _, _ = om.adamw_update(th1, g2, m1, v1, 2, cfg, decay=False)
    b1, b2 = cfg.beta1, cfg.beta2
    for i in range(4):   # scalar arithmetic by hand
        m = b1 * (1 - b1) * g[i] + (1 - b1) * g2[i]
        v = b2 * (1 - b2) * g[i] ** 2 + (1 - b2) * g2[i] ** 2
        upd = (m / (1 - b1 ** 2)) / (math.sqrt(v / (1 - b2 ** 2)) + cfg.adam_eps)
        assert abs(th2[i] - (th1[i] - cfg.lr * upd)) <= 1e-15


def test_microbatch_permutation_invariance():
    cfg = micro_cfg()
    params = micro_params(cfg)
    toks = synth.tokens(4, 1, cfg.seq, cfg.vocab, step=7)
    l1, g1 = om.loss_and_grads(params, toks, cfg)
    l2, g2 = om.loss_and_grads(params, toks[[2, 0, 3, 1]], cfg)
    assert abs(l1 - l2) <= 1e-14 * abs(l1)
    np.testing.assert_allclose(flat(g1), flat(g2), rtol=1e-11, atol=1e-16)
    # gradient of the global mean = weighted sum of per-micro-batch gradient sums
    parts = [om.loss_and_grads(params, toks[i:i + 1], cfg) for i in range(4)]
    np.testing.assert_allclose(l1, np.mean([p[0] for p in parts]), rtol=1e-14)
    np.testing.assert_allclose(flat(g1), sum(flat(p[1]) for p in parts) / 4, rtol=1e-10, atol=1e-16)


def test_model_sizes_match_paper():
    """PAPER.md:202 "668 million to 10 billion" (tests/golden/model_sizes.txt)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "model_sizes.txt")
    with open(path) as fh:
        lines = fh.readlines()
    for line in lines:
        if line.startswith("#") or not line.strip():
            continue
        L, H, V, n = map(int, line.split())
        assert L * 12 * H * H + 2 * V * H == n
    assert abs(669515776 / 668e6 - 1) < 0.003 and abs(9925820416 / 10e9 - 1) < 0.01
    # exact φ = 4H² + 3HI + 2H reduces to 12H² + 2H when I = 8H/3 (H = 96, I = 256)
    cfg = om.ModelConfig(n_layers=1, hidden=96, heads=1, ffn=256, vocab=2, seq=1)
    assert om.phi(cfg) == 12 * 96 * 96 + 2 * 96


def test_attention_row_block_and_key_row_forms_equal_matrix_form():
    """oracle.attention_fwd_rows (a block of query rows) and oracle.attention_key_row (one key row of the backward,
    used for the full-size dK / dV spot checks) agree with the pinned matrix forms; and independently of them the
    key-row form satisfies the identities of the mathematics: Σ_j dK_j = 0 (each row of dS sums to
    Σ_j P_ij dP_ij − δ_i = do_i·o_i − δ_i = 0), Σ_j dV_j = Σ_i do_i (rows of P sum to 1), and the last key is seen
    by the last query only: dV_{S−1} = P_{S−1,S−1}·do_{S−1}."""
    rng = np.random.default_rng(5)
    S, nh, dh = 11, 2, 8
    q, k, v, do = (rng.standard_normal((S, nh, dh)) for _ in range(4))
    o, P = om.attention_fwd(q, k, v)
    _, dk, dv = om.attention_bwd(do, q, k, v, o, P)
    for h in range(nh):
        ob, lb = om.attention_fwd_rows(3, 9, q[:, h], k[:, h], v[:, h])
        np.testing.assert_allclose(ob, o[3:9, h], rtol=1e-12, atol=1e-14)
        o_all, lse_all = om.attention_fwd_rows(0, S, q[:, h], k[:, h], v[:, h])
        for i in (0, 4, S - 1):
            _, lse_i, _ = om.attention_row(i, q[i, h], k[:, h], v[:, h], do[i, h])
            assert abs(lse_all[i] - lse_i) < 1e-12
        sk, sv = np.zeros(dh), np.zeros(dh)
        for j in range(S):
            dkj, dvj = om.attention_key_row(j, k[j, h], v[j, h], q[:, h], do[:, h], o_all, lse_all)
            np.testing.assert_allclose(dkj, dk[j, h], rtol=1e-11, atol=1e-13)
            np.testing.assert_allclose(dvj, dv[j, h], rtol=1e-11, atol=1e-13)
            sk += dkj
            sv += dvj
        np.testing.assert_allclose(sk, 0.0, atol=1e-12)
        np.testing.assert_allclose(sv, do[:, h].sum(0), rtol=1e-12, atol=1e-12)
        _, dv_last = om.attention_key_row(S - 1, k[S - 1, h], v[S - 1, h], q[:, h], do[:, h], o_all, lse_all)
        p_last = np.exp(q[S - 1, h] @ k[S - 1, h] / np.sqrt(dh) - lse_all[S - 1])
        np.testing.assert_allclose(dv_last, p_last * do[S - 1, h], rtol=1e-13)
