"""Per-op parity on a B200 through the kernel-level C ABI (include/tawpipe.h): every HBM-bound kernel and fused
epilogue the training step launches -- RMSNorm forward/backward (every H branch, including the H = 4096 row
kernels C3 runs), RoPE both directions, SwiGLU (separate kernels and the GEMM epilogues the bf16 step uses), the
fused cross-entropy at V = 32000, the deterministic embedding backward and the grouped fp32-accumulate + AdamW of
a9 -- against the fp64 oracle's per-op functions (oracle/model.py) on the same (dtype-rounded) inputs.

Tolerances: fp32 path 1e-5 (outputs) / 1e-6 (AdamW θ, north_star's "≤1e-6 on identical fp32 gradients"); bf16
outputs 1e-2 of the tensor's max (one bf16 rounding is 2^-9 relative; fp32 statistics inside); fp32 outputs of bf16
inputs (rstd, dγ, loss rows) 1e-4.  Errors are max|got − ref| / max|ref| unless stated."""
import numpy as np
import pytest

from helpers import om

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F32, BF = 0, 1


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_09741_b200 import tawpipe
    tawpipe.lib()
    return tawpipe


def tdt(dtype):
    return torch.float32 if dtype == F32 else torch.bfloat16


def dev(a, dtype):
    """numpy -> device tensor of the path's dtype, plus the fp64 copy of exactly what the device holds."""
    t = torch.tensor(np.asarray(a, np.float32)).to(tdt(dtype)).cuda()
    return t, t.double().cpu().numpy()


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def tol(dtype):
    return 1e-5 if dtype == F32 else 1e-2


# ---------------------------------------------------------------------------------------------- RMSNorm
RMS_CASES = [(F32, 37, 64), (F32, 300, 256), (BF, 37, 256), (BF, 70, 1024), (BF, 33, 2048), (BF, 200, 4096),
             (BF, 19, 5120), (BF, 45, 320)]   # bf16: warp-per-row (256, 1024), CTA-per-row (2048, 4096, 5120), generic


@pytest.mark.parametrize("dtype,rows,H", RMS_CASES)
def test_rmsnorm_fwd_bwd_matches_oracle(T, dtype, rows, H):
    rng = np.random.default_rng(rows * 7 + H)
    x, x64 = dev(rng.standard_normal((rows, H)) * 1.5, dtype)
    g, g64 = dev(1.0 + 0.1 * rng.uniform(-1, 1, H), dtype)
    dy, dy64 = dev(rng.standard_normal((rows, H)), dtype)
    res, res64 = dev(rng.standard_normal((rows, H)), dtype)
    eps = 1e-5
    y = torch.empty_like(x)
    rstd = torch.empty(rows, dtype=torch.float32, device="cuda")
    T.rmsnorm_fwd(dtype, rows, H, x.data_ptr(), g.data_ptr(), eps, y.data_ptr(), rstd.data_ptr())
    ry, rr = om.rmsnorm_fwd(x64, g64, eps)
    assert rel(host(y), ry) < tol(dtype)
    assert rel(host(rstd), rr[:, 0]) < 1e-5
    for with_res in (False, True):
        dx = torch.empty_like(x)
        dg = torch.full((H,), 0.5, dtype=torch.float32, device="cuda")    # accumulates into what is there
        T.rmsnorm_bwd(dtype, rows, H, dy.data_ptr(), x.data_ptr(), g.data_ptr(), rstd.data_ptr(),
                      res.data_ptr() if with_res else None, dx.data_ptr(), dg.data_ptr())
        # the oracle's backward on its own r (not the device's rstd): the device rstd is checked above
        rdx, rdg = om.rmsnorm_bwd(dy64, x64, g64, rr)
        if with_res:
            rdx = rdx + res64
        assert rel(host(dx), rdx) < tol(dtype), (with_res, rel(host(dx), rdx))
        assert rel(host(dg) - 0.5, rdg) < (1e-5 if dtype == F32 else 1e-4)


@pytest.mark.parametrize("dtype", [F32, BF])
def test_empty_inputs_are_no_ops(T, dtype):
    """Edge case: zero rows / tokens launch nothing and leave every output untouched (no invalid empty grid)."""
    H, V = 256, 512
    tdt = torch.float32 if dtype == F32 else torch.bfloat16
    x = torch.ones(4, H, dtype=tdt, device="cuda")
    g = torch.ones(H, dtype=tdt, device="cuda")
    y = torch.full((4, H), 3.0, dtype=tdt, device="cuda")
    rstd = torch.full((4,), 5.0, device="cuda")
    T.rmsnorm_fwd(dtype, 0, H, x.data_ptr(), g.data_ptr(), 1e-5, y.data_ptr(), rstd.data_ptr())
    dg = torch.full((H,), 0.5, device="cuda")
    T.rmsnorm_bwd(dtype, 0, H, x.data_ptr(), x.data_ptr(), g.data_ptr(), rstd.data_ptr(), None, y.data_ptr(),
                  dg.data_ptr())
    z = torch.full((4, V), 2.0, dtype=tdt, device="cuda")
    tg = torch.zeros(4, dtype=torch.int32, device="cuda")
    lr = torch.full((4,), 7.0, device="cuda")
    T.cross_entropy(dtype, 0, V, z.data_ptr(), tg.data_ptr(), 1.0, lr.data_ptr())
    E = torch.ones(V, H, dtype=tdt, device="cuda")
    T.embed_fwd(dtype, 1, 0, tg.data_ptr(), 1, E.data_ptr(), H, y.data_ptr())
    torch.cuda.synchronize()
    assert torch.all(y == 3.0) and torch.all(rstd == 5.0) and torch.all(dg == 0.5)
    assert torch.all(z == 2.0) and torch.all(lr == 7.0)


@pytest.mark.parametrize("dtype,rows,H", [(BF, 32768, 4096), (F32, 1000, 96)])   # v8 chunk path / generic path
def test_rmsnorm_bwd_dgamma_is_bit_reproducible(T, dtype, rows, H):
    """dγ's row-block partial sums are added in block order (no atomics): two runs give identical bits."""
    rng = np.random.default_rng(rows + H)
    x, _ = dev(rng.standard_normal((rows, H)), dtype)
    g, _ = dev(1.0 + 0.1 * rng.uniform(-1, 1, H), dtype)
    dy, _ = dev(rng.standard_normal((rows, H)), dtype)
    y = torch.empty_like(x)
    rstd = torch.empty(rows, dtype=torch.float32, device="cuda")
    T.rmsnorm_fwd(dtype, rows, H, x.data_ptr(), g.data_ptr(), 1e-5, y.data_ptr(), rstd.data_ptr())
    outs = []
    for _ in range(2):
        dx = torch.empty_like(x)
        dg = torch.zeros(H, dtype=torch.float32, device="cuda")
        T.rmsnorm_bwd(dtype, rows, H, dy.data_ptr(), x.data_ptr(), g.data_ptr(), rstd.data_ptr(), None,
                      dx.data_ptr(), dg.data_ptr())
        outs.append(host(dg))
    assert np.array_equal(outs[0], outs[1])


# ---------------------------------------------------------------------------------------------- RoPE
@pytest.mark.parametrize("dtype,B,S,nh,dh", [(F32, 2, 200, 3, 64), (F32, 1, 128, 2, 16), (BF, 1, 384, 4, 128),
                                             (BF, 2, 256, 32, 128), (BF, 1, 256, 4, 64), (BF, 1, 64, 2, 32)])
def test_rope_both_directions_match_oracle(T, dtype, B, S, nh, dh):
    rng = np.random.default_rng(S + nh)
    H = nh * dh
    qkv, qkv64 = dev(rng.standard_normal((B * S, 3 * H)), dtype)
    theta = 10000.0
    cos, sin = om.rope_tables(S, dh, theta)
    for inverse in (False, True):
        t = qkv.clone()
        T.rope(dtype, B, S, nh, dh, theta, t.data_ptr(), inverse)
        got = host(t)
        for b in range(B):
            r = slice(b * S, (b + 1) * S)
            for blk in (0, 1):   # q, k rotated
                x = qkv64[r, blk * H:(blk + 1) * H].reshape(S, nh, dh)
                ref = (om.rope_bwd if inverse else om.rope_fwd)(x, cos, sin).reshape(S, H)
                assert rel(got[r, blk * H:(blk + 1) * H], ref) < tol(dtype), (b, blk, inverse)
        assert np.array_equal(got[:, 2 * H:], qkv64[:, 2 * H:])   # v untouched, bit for bit


# ---------------------------------------------------------------------------------------------- SwiGLU
@pytest.mark.parametrize("dtype,rows,I", [(F32, 100, 192), (BF, 300, 768), (BF, 7, 11008)])
def test_swiglu_kernels_match_oracle(T, dtype, rows, I):
    rng = np.random.default_rng(rows + I)
    gu, gu64 = dev(rng.standard_normal((rows, 2 * I)) * 2, dtype)
    dy, dy64 = dev(rng.standard_normal((rows, I)), dtype)
    y = torch.empty((rows, I), dtype=tdt(dtype), device="cuda")
    T.swiglu_fwd(dtype, rows, I, gu.data_ptr(), y.data_ptr())
    u, w = gu64[:, :I], gu64[:, I:]
    assert rel(host(y), om.swiglu_fwd(u, w)) < tol(dtype)
    dgu = torch.empty_like(gu)
    T.swiglu_bwd(dtype, rows, I, dy.data_ptr(), gu.data_ptr(), dgu.data_ptr())
    du, dw = om.swiglu_bwd(dy64, u, w)
    got = host(dgu)
    assert rel(got[:, :I], du) < tol(dtype) and rel(got[:, I:], dw) < tol(dtype)


@pytest.mark.parametrize("M,I,K", [(256, 384, 256), (128, 256, 128), (512, 1024, 512)])   # CTA pair / single CTA
def test_gemm_swiglu_forward_epilogue_matches_oracle(T, M, I, K):
    rng = np.random.default_rng(M + I + K)
    x, x64 = dev(rng.standard_normal((M, K)), BF)
    wgu, w64 = dev(rng.standard_normal((2 * I, K)) / np.sqrt(K) * 2, BF)
    gu = torch.empty((M, 2 * I), dtype=torch.bfloat16, device="cuda")
    y = torch.empty((M, I), dtype=torch.bfloat16, device="cuda")
    T.gemm_swiglu(M, I, K, x.data_ptr(), wgu.data_ptr(), gu.data_ptr(), y.data_ptr())
    ref_gu = x64 @ w64.T
    assert rel(host(gu), ref_gu) < 1e-2
    assert rel(host(y), om.swiglu_fwd(ref_gu[:, :I], ref_gu[:, I:])) < 1e-2
    y2 = torch.empty_like(y)   # gu not stored (the forward of a checkpointed layer): same y
    T.gemm_swiglu(M, I, K, x.data_ptr(), wgu.data_ptr(), None, y2.data_ptr())
    assert torch.equal(y, y2)


@pytest.mark.parametrize("M,I,K", [(256, 384, 256), (512, 512, 512), (128, 256, 128)])
def test_gemm_swiglu_backward_epilogue_matches_oracle(T, M, I, K):
    rng = np.random.default_rng(M * I + K)
    dh, dh64 = dev(rng.standard_normal((M, K)), BF)
    wd, wd64 = dev(rng.standard_normal((K, I)) / np.sqrt(K), BF)     # W_down [H, I]
    gu, gu64 = dev(rng.standard_normal((M, 2 * I)) * 2, BF)
    dgu = torch.empty((M, 2 * I), dtype=torch.bfloat16, device="cuda")
    T.gemm_swiglu_bwd(M, I, K, dh.data_ptr(), wd.data_ptr(), gu.data_ptr(), dgu.data_ptr())
    dY = dh64 @ wd64                                                  # dy = dh2·W_down
    du, dw = om.swiglu_bwd(dY, gu64[:, :I], gu64[:, I:])
    got = host(dgu)
    assert rel(got[:, :I], du) < 1e-2 and rel(got[:, I:], dw) < 1e-2


# ---------------------------------------------------------------------------------------------- cross-entropy
@pytest.mark.parametrize("dtype,rows,V", [(F32, 67, 512), (BF, 300, 32000), (BF, 1, 128)])
def test_cross_entropy_matches_oracle(T, dtype, rows, V):
    rng = np.random.default_rng(rows + V)
    z, z64 = dev(rng.standard_normal((rows, V)) * 3, dtype)
    tgt = rng.integers(0, V, rows).astype(np.int32)
    tgt[0] = V - 1
    tg = torch.tensor(tgt).cuda()
    loss = torch.empty(rows, dtype=torch.float32, device="cuda")
    denom = 1234.0
    T.cross_entropy(dtype, rows, V, z.data_ptr(), tg.data_ptr(), 1.0 / denom, loss.data_ptr())
    dz = host(z)
    lr = host(loss)
    for r in range(rows):
        l_r, dz_r = om.cross_entropy_fwd_bwd(z64[r:r + 1], tgt[r:r + 1], denom)
        assert abs(lr[r] - l_r) <= (1e-5 if dtype == F32 else 1e-4) * max(1.0, abs(l_r)), (r, lr[r], l_r)
        assert np.max(np.abs(dz[r] - dz_r[0])) <= tol(dtype) * np.max(np.abs(dz_r)), r


# ---------------------------------------------------------------------------------------------- embedding
@pytest.mark.parametrize("dtype,B,S,V,H", [(F32, 2, 300, 1000, 64), (BF, 2, 300, 1000, 256), (BF, 1, 2048, 32000, 4096)])
def test_embedding_fwd_and_deterministic_bwd_match_oracle(T, dtype, B, S, V, H):
    rng = np.random.default_rng(V + S)
    tok = ((rng.zipf(1.1, (B, S + 1)) - 1) % V).astype(np.int32)   # Zipf: long segments for frequent tokens
    tok[0, :50] = 3                                                  # one token at 50 consecutive positions
    tk = torch.tensor(tok).cuda()
    E, E64 = dev(rng.standard_normal((V, H)) * 0.02, dtype)
    h = torch.empty((B * S, H), dtype=tdt(dtype), device="cuda")
    T.embed_fwd(dtype, B, S, tk.data_ptr(), S + 1, E.data_ptr(), H, h.data_ptr())
    x = tok[:, :S].reshape(-1)
    assert np.array_equal(host(h), E64[x])
    dh, dh64 = dev(rng.standard_normal((B * S, H)), dtype)
    outs = []
    for _ in range(2):
        dE = torch.full((V, H), 0.25, dtype=torch.float32, device="cuda")
        T.embed_bwd(dtype, B, S, tk.data_ptr(), S + 1, dh.data_ptr(), H, V, dE.data_ptr())
        outs.append(host(dE))
    assert np.array_equal(outs[0], outs[1])                        # bit-reproducible
    ref = np.zeros((V, H))
    np.add.at(ref, x, dh64)                                          # dE[x_p] += dh0[p] (oracle/model.py)
    assert rel(outs[0] - 0.25, ref) < 1e-5
    untouched = np.setdiff1d(np.arange(V), x)
    assert np.all(outs[0][untouched] == 0.25)


# ---------------------------------------------------------------------------------------------- rail partial (a8)
@pytest.mark.parametrize("wdt,G,n", [(F32, 1, 4096), (F32, 2, 1000), (BF, 2, 65536), (BF, 4, 12288), (F32, 8, 4100)])
def test_group_partial_matches_member_order_sum(T, wdt, G, n):
    """a8 on the peer path: a non-owner group's rail partial is the members' fp32 stripes summed in member order
    (R16, oracle/schedule.py reduce: acc = acc + piece, jj ascending), cast once to the wire dtype."""
    rng = np.random.default_rng(G * 1000 + n)
    xs = [(rng.standard_normal(n) * 10.0 ** rng.integers(-3, 1)).astype(np.float32) for _ in range(G)]
    srcs = [torch.tensor(x).cuda() for x in xs]
    tdt = torch.float32 if wdt == F32 else torch.bfloat16
    out = torch.full((n,), 9.0, dtype=tdt, device="cuda")
    T.group_partial(wdt, [t.data_ptr() for t in srcs], n, out.data_ptr())
    torch.cuda.synchronize()
    acc = xs[0].copy()
    for x in xs[1:]:
        acc = (acc + x).astype(np.float32)   # fp32, member order: the kernel's exact arithmetic
    want = torch.tensor(acc).to(tdt)            # one round-to-nearest-even cast to the wire dtype
    assert torch.equal(out.cpu(), want)
    ref64 = np.sum(np.stack(xs).astype(np.float64), axis=0)   # the oracle's fp64 sum
    assert rel(out.float().cpu().numpy(), ref64) < (1e-6 if wdt == F32 else 1e-2)


# ---------------------------------------------------------------------------------------------- AdamW (a9)
ADAM_CASES = [
    # (name, wire dtype, n, groups as lists of source dtypes, eps, wd)
    ("p1", F32, 4096, [["f32"]], 1e-8, 0.1),
    ("g2-fp32", F32, 1000, [["f32", "f32"]], 1e-8, 0.1),                       # scalar path (n % 8 != 0)
    ("d2-bf16", BF, 8192, [["f32"], ["bf16"]], 1e-8, 0.1),
    ("d4g2-owner1", BF, 12288, [["bf16"], ["f32", "f32"], ["bf16"], ["bf16"]], 1e-8, 0.1),   # owner group 1 of 4
    ("d3g3", BF, 4160, [["bf16"], ["bf16"], ["f32", "f32", "f32"]], 1.0, 0.0),  # eps ≫ |g|: Δ ∝ g
    ("g4-eps1", F32, 2048, [["f32", "f32", "f32", "f32"]], 1.0, 0.0),
]


@pytest.mark.parametrize("name,wdt,n,groups,eps,wd", ADAM_CASES, ids=[c[0] for c in ADAM_CASES])
def test_grouped_accumulate_adamw_matches_oracle(T, name, wdt, n, groups, eps, wd):
    rng = np.random.default_rng(n + len(groups))
    theta0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    master = torch.tensor(theta0).cuda()
    m = torch.zeros(n, dtype=torch.float32, device="cuda")
    v = torch.zeros(n, dtype=torch.float32, device="cuda")
    wire = torch.empty(n, dtype=tdt(wdt), device="cuda")
    nd = (100, 300, n - 64, n)   # two no-decay ranges (RMSNorm gains), unit_off 37
    unit_off = 37
    pos = unit_off + np.arange(n)
    decay = ~(((pos >= nd[0]) & (pos < nd[1])) | ((pos >= nd[2]) & (pos < nd[3])))
    # ε ≫ |g| cases run at lr = 1 (update ≈ −m̂, well above the fp32 resolution of θ)
    cfg = om.ModelConfig(n_layers=1, hidden=8, heads=1, ffn=8, vocab=8, seq=1, lr=1.0 if eps >= 1e-3 else 1e-3,
                         adam_eps=eps, weight_decay=wd)
    th_r, m_r, v_r = theta0.astype(np.float64), np.zeros(n), np.zeros(n)
    prev = theta0.astype(np.float64)
    for step in (1, 2, 3):
        srcs, keep, g_ref = [], [], np.zeros(n)
        for gr in groups:
            part = np.zeros(n)
            row = []
            for kind in gr:
                a = rng.standard_normal(n) * 1e-3 * (1 + step)
                t, a64 = dev(a, F32 if kind == "f32" else wdt)
                keep.append(t)
                row.append((t.data_ptr(), kind == "f32"))
                part += a64
            g_ref += part
            srcs.append(row)
        T.adamw(wdt, srcs, master.data_ptr(), m.data_ptr(), v.data_ptr(), wire.data_ptr(), n, unit_off, nd,
                lr=cfg.lr, eps=eps, wd=wd, step=step)
        torch.cuda.synchronize()
        # oracle: AdamW on the exact sum of the same inputs, element by element by decay class
        th_new = np.empty(n)
        for dc in (True, False):
            sel = decay == dc
            th_new[sel], m_r[sel], v_r[sel] = om.adamw_update(th_r[sel], g_ref[sel], m_r[sel], v_r[sel], step, cfg, dc)
        d_ref = th_new - th_r
        got = host(master)
        assert np.max(np.abs(got - th_new)) <= 1e-6 * np.max(np.abs(th_new)), (step, rel(got, th_new))
        # the update itself, per element relative to the largest update (catches a wrong group sum or scale)
        d_got = got - prev
        assert np.max(np.abs(d_got - d_ref)) <= 1e-4 * np.max(np.abs(d_ref)), (step, np.max(np.abs(d_got - d_ref)))
        prev = got
        assert rel(host(m), m_r) < 1e-5 and rel(host(v), v_r) < 1e-5
        assert torch.equal(wire, master.to(tdt(wdt)))   # the wire copy is the rounded master, bit for bit
        th_r = th_new


@pytest.mark.parametrize("M,H,nh,S", [(512, 256, 2, 256), (256, 512, 8, 128), (1024, 1024, 8, 512)])
def test_gemm_rope_epilogue_matches_oracle(T, M, H, nh, S):
    """QKV projection with RoPE in the tcgen05 epilogue (the bf16 step's path): q | k columns of x·Wᵀ rotated as
    oracle.rope_fwd, v columns plain; M rows are M // S sequences (p = row mod S); CTA-pair (N % 256 == 0) shapes."""
    dh = H // nh
    rng = np.random.default_rng(M + H)
    x, x64 = dev(rng.standard_normal((M, H)), BF)
    w, w64 = dev(rng.standard_normal((3 * H, H)) / np.sqrt(H), BF)
    qkv = torch.empty((M, 3 * H), dtype=torch.bfloat16, device="cuda")
    T.gemm_rope(M, 3 * H, H, x.data_ptr(), w.data_ptr(), qkv.data_ptr(), S, dh, 10000.0, 2 * H)
    got = host(qkv)
    ref = x64 @ w64.T
    cos, sin = om.rope_tables(S, dh, 10000.0)
    for b in range(M // S):
        r = slice(b * S, (b + 1) * S)
        for blk in (0, 1):
            rr = om.rope_fwd(ref[r, blk * H:(blk + 1) * H].reshape(S, nh, dh), cos, sin).reshape(S, H)
            assert rel(got[r, blk * H:(blk + 1) * H], rr) < 1e-2, (b, blk)
    assert rel(got[:, 2 * H:], ref[:, 2 * H:]) < 1e-2
