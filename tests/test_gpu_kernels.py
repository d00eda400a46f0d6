"""Reduction / elementwise kernels of libnnt vs the oracle (element by element).

maxsumexp + softmax including per-key-tile accumulate calls and the
causal extents; softmax backward; LayerNorm fwd/bwd; GELU; bias-grad
column sums; Adam; dot / scale.
"""
import math

import numpy as np
import pytest
import torch

import nnt_inputs
from oracle import dense, tiled
from gpu_util import close, close_update, bf16_round, dev, host, rel

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import nnt


def _scores(rows, cols, seed, scale=4.0):
    rng = np.random.default_rng(seed)
    return (scale * rng.standard_normal((rows, cols))).astype(np.float32)


def _mask(rows, cols, seq_q, causal):
    if not causal:
        return np.ones((rows, cols), bool)
    q = (np.arange(rows) % seq_q)[:, None]
    return np.arange(cols)[None, :] <= q


@pytest.mark.parametrize("causal", [0, 1])
@pytest.mark.parametrize("cols,tile_k", [(1024, 1024), (1024, 96), (32, 16), (520, 200), (2048, 512)])
def test_maxsumexp_and_softmax(causal, cols, tile_k):
    seq_q = cols
    rows = 3 * seq_q if cols <= 1024 else seq_q
    x = _scores(rows, cols, seed=cols + tile_k)
    X = dev(x)
    st = torch.zeros(rows, 2, device="cuda")
    nnt.nnt_maxsumexp(X, rows, cols, cols, tile_k, causal, seq_q, st)
    mask = _mask(rows, cols, seq_q, causal)
    m_ref, s_ref = dense.maxsumexp(x.astype(np.float64), mask)
    got = host(st)
    assert np.array_equal(got[:, 0], m_ref.astype(np.float32))  # the max is exact
    close(got[:, 1], s_ref, 1e-5)
    for ydt in ("f32", "bf16"):
        Y = torch.full((rows, cols), float("nan"), device="cuda",
                       dtype=torch.float32 if ydt == "f32" else torch.bfloat16)
        nnt.nnt_softmax(X, rows, cols, cols, tile_k, causal, seq_q, st, Y, 0 if ydt == "f32" else 1, cols)
        torch.cuda.synchronize()
        p_ref = dense.softmax(x.astype(np.float64), mask)
        y = host(Y)
        if causal:
            q = np.arange(rows) % seq_q
            extent = np.minimum(cols, ((q + 1 + 127) // 128) * 128)
            written = np.arange(cols)[None, :] < extent[:, None]
            assert np.all(np.isfinite(y[written])) and np.all(np.isnan(y[~written]))
            assert np.all(y[written & ~mask] == 0.0)
            y = np.where(written, y, 0.0)
        tol = 1e-5 if ydt == "f32" else 4e-3
        close(y, p_ref, tol)
        if ydt == "f32":
            np.testing.assert_allclose(y.sum(-1), 1.0, atol=1e-5)


def test_maxsumexp_accumulate_per_key_tile_equals_single_call():
    """The paper's first subroutine called once per key tile with Reduce (accumulate) semantics."""
    rows, cols, seq_q = 256, 1024, 256
    x = _scores(rows, cols, seed=3, scale=10.0)
    X = dev(x)
    st1 = torch.zeros(rows, 2, device="cuda")
    nnt.nnt_maxsumexp(X, rows, cols, cols, cols, 0, seq_q, st1)
    st2 = torch.zeros(rows, 2, device="cuda")
    for j, k0 in enumerate(range(0, cols, 256)):
        nnt.nnt_maxsumexp(X.data_ptr() + 4 * k0, rows, 256, cols, 256, 0, seq_q, st2, accumulate=int(j > 0))
    torch.cuda.synchronize()
    a, b = host(st1), host(st2)
    assert np.array_equal(a[:, 0], b[:, 0])
    close(b[:, 1], a[:, 1], 1e-6)


def test_softmax_large_logits_no_nan():
    x = np.array([[1000.0, 0.0, 0.0, 0.0], [-1000.0, -1000.0, -1000.0, -1000.0]], np.float32)
    X = dev(x)
    st = torch.zeros(2, 2, device="cuda")
    Y = torch.zeros(2, 4, device="cuda")
    nnt.nnt_maxsumexp(X, 2, 4, 4, 4, 0, 2, st)
    nnt.nnt_softmax(X, 2, 4, 4, 4, 0, 2, st, Y, 0, 4)
    y = host(Y)
    assert np.array_equal(y[0], [1.0, 0.0, 0.0, 0.0])
    np.testing.assert_allclose(y[1], 0.25, rtol=1e-6)


@pytest.mark.parametrize("causal", [0, 1])
@pytest.mark.parametrize("pdt", ["f32", "bf16"])
def test_softmax_bwd(causal, pdt):
    rows, cols, seq_q = 512, 256, 256
    x = _scores(rows, cols, seed=9)
    mask = _mask(rows, cols, seq_q, causal)
    p = dense.softmax(x.astype(np.float64), mask)
    if pdt == "bf16":
        p = bf16_round(p)
    dp = _scores(rows, cols, seed=10, scale=1.0)
    dp_dev = dev(dp)
    if causal:  # dP above the diagonal is never read: poison it
        dp_dev = dev(np.where(mask, dp, np.nan).astype(np.float32))
    P = dev(p, torch.float32 if pdt == "f32" else torch.bfloat16)
    DA = torch.full((rows, cols), float("nan"), device="cuda",
                    dtype=torch.float32 if pdt == "f32" else torch.bfloat16)
    code = 0 if pdt == "f32" else 1
    scale = 0.125
    nnt.nnt_softmax_bwd(P, code, cols, dp_dev, cols, rows, cols, causal, seq_q, scale, DA, code, cols)
    torch.cuda.synchronize()
    want = scale * dense.softmax_bwd(p, np.where(mask, dp, 0.0))
    got = host(DA)
    if causal:
        q = np.arange(rows) % seq_q
        extent = np.minimum(cols, ((q + 1 + 127) // 128) * 128)
        written = np.arange(cols)[None, :] < extent[:, None]
        assert np.all(got[written & ~mask] == 0.0)
        got = np.where(written, got, 0.0)
    close(got, want, (1e-5 if pdt == "f32" else 4e-3))


# E <= 1024: warp per row; 1024 < E <= 2048: 4-warp groups striding over rows with the next row
# prefetched (T = 5000: several rows per group, ragged last stride); above: one CTA per row
@pytest.mark.parametrize("E,T", [(64, 96), (768, 96), (1028, 5000), (1600, 96), (1600, 5000), (2048, 5000),
                                 (2052, 96), (8192, 96)])
@pytest.mark.parametrize("ydt", ["f32", "bf16"])
@pytest.mark.parametrize("ring", ["0", "1"])
def test_layernorm_fwd(E, T, ydt, ring, monkeypatch):
    monkeypatch.setenv("NNT_LN_FWD_RING", ring)  # 1024 < E <= 2048: also the (opt-in) ring kernel
    rng = np.random.default_rng(E)
    x = (50.0 + 3.0 * rng.standard_normal((T, E))).astype(np.float32)  # |mean| >> std
    g = (1 + 0.1 * rng.standard_normal(E)).astype(np.float32)
    b = (0.1 * rng.standard_normal(E)).astype(np.float32)
    Y = torch.zeros(T, E, device="cuda", dtype=torch.float32 if ydt == "f32" else torch.bfloat16)
    mean = torch.zeros(T, device="cuda")
    rstd = torch.zeros(T, device="cuda")
    nnt.nnt_layernorm_fwd(dev(x), T, E, E, 1024, dev(g), dev(b), 1e-5, Y, 0 if ydt == "f32" else 1, E, mean, rstd)
    torch.cuda.synchronize()
    y_ref, m_ref, r_ref = dense.layernorm_fwd(x, g, b, 1e-5)
    close(host(Y), y_ref, (2e-5 if ydt == "f32" else 4e-3))
    close(host(mean), m_ref, 1e-6)
    close(host(rstd), r_ref, 1e-4)


def test_layernorm_closed_forms():
    """Constant rows -> beta; [1,3,...] pattern -> +-1/sqrt(1+eps) (tests/golden/layernorm_spec.json)."""
    E = 64
    x = np.zeros((2, E), np.float32)
    x[0] = 3.5
    x[1, 0::2], x[1, 1::2] = 1.0, 3.0
    g = np.ones(E, np.float32)
    b = np.linspace(-1, 1, E).astype(np.float32)
    Y = torch.zeros(2, E, device="cuda")
    mean, rstd = torch.zeros(2, device="cuda"), torch.zeros(2, device="cuda")
    nnt.nnt_layernorm_fwd(dev(x), 2, E, E, 16, dev(g), dev(b), 1e-5, Y, 0, E, mean, rstd)
    y = host(Y)
    np.testing.assert_allclose(y[0], b, atol=1e-6)
    v = 1 / math.sqrt(1 + 1e-5)
    np.testing.assert_allclose(y[1] - b, np.where(np.arange(E) % 2 == 0, -v, v), rtol=1e-6)


# E <= 1024: the warp-per-row kernel; 1024 < E <= 2048: 4-warp groups fed by shared-memory row rings
# (bulk copies, 4 rows ahead); above: warp groups (8 warps), the next row prefetched in registers up
# to E = 4096.  T = 8192 gives several rows per group.
@pytest.mark.parametrize("E,T", [(64, 200), (768, 200), (1028, 3000), (1280, 200), (1600, 200), (1600, 8192),
                                 (2048, 2000), (2052, 300), (4096, 200), (8192, 100)])
def test_layernorm_bwd(E, T):
    rng = np.random.default_rng(E + 1)
    x = (1.0 + 2.0 * rng.standard_normal((T, E))).astype(np.float32)
    g = (1 + 0.1 * rng.standard_normal(E)).astype(np.float32)
    b = np.zeros(E, np.float32)
    dy = rng.standard_normal((T, E)).astype(np.float32)
    dres = rng.standard_normal((T, E)).astype(np.float32)
    _, m_ref, r_ref = dense.layernorm_fwd(x, g, b, 1e-5)
    dx_ref, dg_ref, db_ref = dense.layernorm_bwd(dy, x, g, m_ref, r_ref)
    DX = torch.zeros(T, E, device="cuda")
    DX16 = torch.zeros(T, E, device="cuda", dtype=torch.bfloat16)
    DG = dev(np.ones(E, np.float32))
    DB = dev(np.ones(E, np.float32))
    nb = nnt.nnt_layernorm_bwd_scratch_bytes(T, E)
    scr = torch.empty(nb, device="cuda", dtype=torch.uint8)
    # the fused column sum of the output dx (every E)
    DS = dev(np.full(E, 2.0, np.float32))
    nnt.nnt_layernorm_bwd(dev(dy), E, dev(x), E, dev(m_ref.astype(np.float32)), dev(r_ref.astype(np.float32)),
                          dev(g), T, E, dev(dres), DX, E, DX16, DG, DB, DS, 1, scr, nb)
    torch.cuda.synchronize()
    close(host(DX), dx_ref + dres, 1e-5)
    close(host(DX16), dx_ref + dres, 4e-3)
    close(host(DG), dg_ref + 1.0, 1e-5)
    close(host(DB), db_ref + 1.0, 1e-5)
    close(host(DS), (dx_ref + dres).sum(axis=0) + 2.0, 1e-5)


@pytest.mark.parametrize("E,extras", [(1600, True), (1600, False), (1028, False), (2048, True)])
def test_layernorm_bwd_ring_equals_group_kernel(E, extras, monkeypatch):
    """1024 < E <= 2048: the ring kernel (rows streamed into shared memory) keeps the group kernel's
    arithmetic -- same row-to-group assignment, column mapping, per-row sum order and column
    partials -- so every output is bitwise equal to NNT_LN_BWD_RING=0's; with and without the
    residual gradient, the bf16 copy and the fused column sum."""
    T = 5000
    rng = np.random.default_rng(E + 7)
    x = (1.0 + 2.0 * rng.standard_normal((T, E))).astype(np.float32)
    g = (1 + 0.1 * rng.standard_normal(E)).astype(np.float32)
    dy = rng.standard_normal((T, E)).astype(np.float32)
    dres = rng.standard_normal((T, E)).astype(np.float32)
    _, m_ref, r_ref = dense.layernorm_fwd(x, g, np.zeros(E, np.float32), 1e-5)
    nb = nnt.nnt_layernorm_bwd_scratch_bytes(T, E)
    args = (dev(dy), E, dev(x), E, dev(m_ref.astype(np.float32)), dev(r_ref.astype(np.float32)), dev(g), T, E)
    R = dev(dres)
    outs = []
    for ring in ("1", "0"):
        monkeypatch.setenv("NNT_LN_BWD_RING", ring)
        DX = torch.zeros(T, E, device="cuda")
        DX16 = torch.zeros(T, E, device="cuda", dtype=torch.bfloat16) if extras else None
        DG, DB = torch.zeros(E, device="cuda"), torch.zeros(E, device="cuda")
        DS = torch.zeros(E, device="cuda") if extras else None
        scr = torch.empty(nb, device="cuda", dtype=torch.uint8)
        nnt.nnt_layernorm_bwd(*args, R if extras else None, DX, E, DX16, DG, DB, DS, 0, scr, nb)
        torch.cuda.synchronize()
        outs.append([host(t) for t in (DX, DX16, DG, DB, DS) if t is not None])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    dx_ref, dg_ref, db_ref = dense.layernorm_bwd(dy, x, g, m_ref, r_ref)
    close(outs[0][0], dx_ref + (dres if extras else 0), 1e-5)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_gelu(dt):
    n = 100003
    x = np.linspace(-8, 8, n).astype(np.float32)
    dy = np.cos(np.arange(n)).astype(np.float32)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    code = 0 if dt == "f32" else 1
    if dt == "bf16":
        x, dy = bf16_round(x), bf16_round(dy)
    X, DY = dev(x, tdt), dev(dy, tdt)
    Y, DX = torch.empty_like(X), torch.empty_like(X)
    nnt.nnt_gelu_fwd(X, Y, code, n)
    nnt.nnt_gelu_bwd(X, DY, DX, code, n)
    torch.cuda.synchronize()
    tol = 1e-6 if dt == "f32" else 4e-3
    close(host(Y), dense.gelu(x), tol)
    close(host(DX), dense.gelu_bwd(x, dy), tol)
    assert host(Y)[n // 2] == 0.0  # gelu(0) = 0


@pytest.mark.parametrize("T,N", [(8192, 768), (1000, 3072), (33, 100)])
def test_bias_grad(T, N):
    rng = np.random.default_rng(T)
    dy = rng.standard_normal((T, N)).astype(np.float32)
    db0 = rng.standard_normal(N).astype(np.float32)
    DB = dev(db0)
    nb = nnt.nnt_bias_grad_scratch_bytes(T, N)
    scr = torch.empty(nb, device="cuda", dtype=torch.uint8)
    C16 = torch.zeros(T, N, device="cuda", dtype=torch.bfloat16)
    nnt.nnt_bias_grad(dev(dy), 0, T, N, N, DB, 1, C16, scr, nb)
    torch.cuda.synchronize()
    close(host(DB), dy.astype(np.float64).sum(0) + db0, 1e-5)
    assert np.array_equal(host(C16), bf16_round(dy))
    # deterministic: bitwise identical on repeat
    DB2 = dev(db0)
    nnt.nnt_bias_grad(dev(dy), 0, T, N, N, DB2, 1, None, scr, nb)
    torch.cuda.synchronize()
    assert torch.equal(DB, DB2)


def test_adam_matches_oracle_and_step1_closed_form():
    n = 10007
    rng = np.random.default_rng(1)
    w = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    W, M, V = dev(w), dev(m), dev(v)
    W16 = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    wr, mr, vr = w.astype(np.float64), m.astype(np.float64), v.astype(np.float64)
    for t in range(1, 4):
        g = rng.standard_normal(n).astype(np.float32)
        hp = nnt.adam_hparams(1e-3, 0.9, 0.999, 1e-8, 0.0, t)
        nnt.nnt_adam_step(n, W, dev(g), M, V, W16, hp)
        wr, mr, vr = dense.adam_step(wr, g, mr, vr, t)
        torch.cuda.synchronize()
        # compare the update, not w; fp32 storage of w ~ N(0,1) bounds the update's rel error
        # near 2^-24 / lr ~ 6e-5 (worst element), hence the fp32-path tolerance
        close_update(host(W) - w, wr - w, wr, np.sqrt(vr), 1e-4)
        # (1 - beta) passed as fp32 roundings of the fp64 values (R23): m and v to fp32 rounding
        close(host(M), mr, 1e-6, "m")
        close(host(V), vr, 1e-6, "v")
        assert np.array_equal(host(W16), bf16_round(host(W)))


def test_adamw_decoupled_decay_matches_oracle():
    """AdamW (weight_decay > 0, decoupled: w -= lr * wd * w_old, reading R12) vs the oracle, which
    is itself pinned to torch.optim.AdamW."""
    n = 4099
    rng = np.random.default_rng(5)
    w = rng.standard_normal(n).astype(np.float32)
    W, M, V = dev(w), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    wr, mr, vr = w.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(1, 4):
        g = rng.standard_normal(n).astype(np.float32)
        hp = nnt.adam_hparams(1e-2, 0.9, 0.999, 1e-8, 0.1, t)
        nnt.nnt_adam_step(n, W, dev(g), M, V, None, hp)
        wr, mr, vr = dense.adam_step(wr, g, mr, vr, t, lr=1e-2, weight_decay=0.1)
        torch.cuda.synchronize()
        close_update(host(W) - w, wr - w, wr, np.sqrt(vr), 1e-4)


def test_sgd_momentum_matches_oracle():
    n = 5003
    rng = np.random.default_rng(6)
    w = rng.standard_normal(n).astype(np.float32)
    W, BUF = dev(w), torch.zeros(n, device="cuda")
    W16 = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    wr, br = w.astype(np.float64), np.zeros(n)
    for t in range(3):
        g = rng.standard_normal(n).astype(np.float32)
        nnt.nnt_sgd_step(n, W, dev(g), BUF, W16, 1e-2, 0.9, 0.01)
        wr, br = dense.sgd_step(wr, g, br, lr=1e-2, momentum=0.9, weight_decay=0.01)
        torch.cuda.synchronize()
        close(host(W) - w, wr - w, 1e-5, "dw")
        close(host(BUF), br, 1e-6, "buf")
        assert np.array_equal(host(W16), bf16_round(host(W)))


def test_dot_and_scale():
    n = 123457
    rng = np.random.default_rng(2)
    y = rng.standard_normal(n).astype(np.float32)
    r = rng.standard_normal(n).astype(np.float32)
    out = torch.zeros(1, device="cuda")
    nb = nnt.nnt_dot_scratch_bytes(n)
    scr = torch.empty(nb, device="cuda", dtype=torch.uint8)
    nnt.nnt_dot(dev(y), dev(r), n, 0.5, out, scr, nb)
    Y = torch.empty(n, device="cuda")
    nnt.nnt_scale(dev(r), 0.25, Y, n)
    torch.cuda.synchronize()
    assert abs(out.item() - 0.5 * float(y.astype(np.float64) @ r)) < 1e-6 * abs(0.5 * float(y @ r)) + 1e-6
    assert np.array_equal(host(Y), (0.25 * r).astype(np.float32))
