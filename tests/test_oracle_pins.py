"""Pins of oracle/dense.py against things other than itself.

Closed forms and worked examples (tests/golden, cited), torch fp64 library
routines for the special cases that reduce to them (F.layer_norm, F.gelu,
F.scaled_dot_product_attention, torch.optim.Adam/AdamW, autograd), central
finite differences, and invariants.  No GPU.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import nnt_inputs
from oracle import dense

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _t(a):
    return torch.tensor(np.asarray(a, np.float64), dtype=torch.float64)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ----------------------------------------------------------------- softmax
def test_softmax_golden():
    for case in _gold("softmax_spec.json")["cases"]:
        p = dense.softmax(np.array(case["t"]))
        assert np.all(np.isfinite(p))
        np.testing.assert_allclose(p, case["p"], rtol=0, atol=1e-15)


def test_softmax_rows_sum_to_one_and_match_torch():
    rng = np.random.default_rng(0)
    t = 5 * rng.standard_normal((7, 13))
    p = dense.softmax(t)
    np.testing.assert_allclose(p.sum(-1), 1.0, atol=1e-15)
    np.testing.assert_allclose(p, torch.softmax(_t(t), -1).numpy(), rtol=1e-14, atol=0)


def test_maxsumexp_definition_and_masked_identity():
    t = np.array([[1.0, 2.0, 3.0], [0.0, 0.0, 0.0]])
    m, s = dense.maxsumexp(t)
    np.testing.assert_allclose(m, [3.0, 0.0])
    np.testing.assert_allclose(s, [math.exp(-2) + math.exp(-1) + 1.0, 3.0], rtol=1e-15)
    m, s = dense.maxsumexp(t, mask=np.zeros_like(t, dtype=bool))
    assert np.all(m == -np.inf) and np.all(s == 0.0)
    # logsumexp identity: m + log(s) == torch.logsumexp
    rng = np.random.default_rng(1)
    t = 30 * rng.standard_normal((4, 50))
    m, s = dense.maxsumexp(t)
    np.testing.assert_allclose(m + np.log(s), torch.logsumexp(_t(t), -1).numpy(), rtol=1e-14)


def test_softmax_bwd_invariants_and_fd():
    rng = np.random.default_rng(2)
    t = rng.standard_normal((3, 9))
    dp = rng.standard_normal((3, 9))
    p = dense.softmax(t)
    da = dense.softmax_bwd(p, dp)
    np.testing.assert_allclose(da.sum(-1), 0.0, atol=1e-15)
    # FD of <softmax(t), dp> w.r.t. t
    h = 1e-6
    fd = np.zeros_like(t)
    for idx in np.ndindex(t.shape):
        tp, tm = t.copy(), t.copy()
        tp[idx] += h
        tm[idx] -= h
        fd[idx] = ((dense.softmax(tp) * dp).sum() - (dense.softmax(tm) * dp).sum()) / (2 * h)
    assert rel(da, fd) < 1e-8


# ----------------------------------------------------------------- GELU
def test_gelu_golden_and_symmetry():
    for c in _gold("gelu_closed_form.json")["cases"]:
        assert abs(dense.gelu(c["u"]) - c["gelu"]) <= 1e-15 * max(1, abs(c["gelu"]))
        if "dgelu" in c:
            assert abs(dense.gelu_grad(c["u"]) - c["dgelu"]) < 1e-15
    x = np.linspace(-6, 6, 101)
    np.testing.assert_allclose(dense.gelu(x) - dense.gelu(-x), x, atol=1e-14)


def test_gelu_vs_torch_tanh_gelu():
    x = np.linspace(-8, 8, 1001)
    xt = _t(x).requires_grad_(True)
    y = F.gelu(xt, approximate="tanh")
    y.sum().backward()
    np.testing.assert_allclose(dense.gelu(x), y.detach().numpy(), rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(dense.gelu_grad(x), xt.grad.numpy(), rtol=1e-13, atol=1e-13)


def test_gelu_grad_fd():
    x = np.linspace(-5, 5, 41)
    h = 1e-6
    fd = (dense.gelu(x + h) - dense.gelu(x - h)) / (2 * h)
    np.testing.assert_allclose(dense.gelu_grad(x), fd, rtol=1e-8, atol=1e-9)


# ----------------------------------------------------------------- LayerNorm
def test_layernorm_golden():
    g = _gold("layernorm_spec.json")
    for c in g["cases"]:
        y, _, _ = dense.layernorm_fwd(np.array(c["x"]), np.array(c["gamma"]), np.array(c["beta"]), g["eps"])
        np.testing.assert_allclose(y, c["y"], rtol=0, atol=1e-15)


def test_layernorm_moments_exact():
    rng = np.random.default_rng(3)
    x = 3.0 + 2.0 * rng.standard_normal((5, 64))
    eps = 1e-5
    y, mu, r = dense.layernorm_fwd(x, np.ones(64), np.zeros(64), eps)
    var = x.var(-1)
    np.testing.assert_allclose(y.mean(-1), 0.0, atol=1e-14)
    # var(xhat) = sigma^2 / (sigma^2 + eps) exactly ("unit variance" up to O(eps/sigma^2))
    np.testing.assert_allclose(y.var(-1), var / (var + eps), rtol=1e-13)


def test_layernorm_vs_torch_and_autograd():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 3, 16)) * 1.7 + 0.3
    g = 1 + 0.1 * rng.standard_normal(16)
    b = 0.1 * rng.standard_normal(16)
    dy = rng.standard_normal(x.shape)
    xt, gt, bt = (_t(a).requires_grad_(True) for a in (x, g, b))
    yt = F.layer_norm(xt, (16,), gt, bt, eps=1e-5)
    (yt * _t(dy)).sum().backward()
    y, mu, r = dense.layernorm_fwd(x, g, b, 1e-5)
    assert rel(y, yt.detach().numpy()) < 1e-14
    dx, dg, db = dense.layernorm_bwd(dy, x, g, mu, r)
    assert rel(dx, xt.grad.numpy()) < 1e-13
    assert rel(dg, gt.grad.numpy()) < 1e-13
    assert rel(db, bt.grad.numpy()) < 1e-13
    # sum_e dx = 0 exactly (LN output is shift-invariant)
    np.testing.assert_allclose(dx.sum(-1), 0.0, atol=1e-13)


# ----------------------------------------------------------------- linear
def test_linear_identity_and_integer_exact():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 6, 8))
    y = dense.linear_fwd(x, np.eye(8), np.zeros(8))
    assert np.array_equal(y, x)
    xi = rng.integers(-4, 5, (5, 7)).astype(float)
    wi = rng.integers(-4, 5, (3, 7)).astype(float)
    bi = rng.integers(-4, 5, 3).astype(float)
    y = dense.linear_fwd(xi, wi, bi)
    brute = np.array([[sum(wi[d, e] * xi[t, e] for e in range(7)) + bi[d] for d in range(3)] for t in range(5)])
    assert np.array_equal(y, brute)


def test_linear_bwd_vs_autograd():
    rng = np.random.default_rng(6)
    x, w, b = rng.standard_normal((2, 5, 7)), rng.standard_normal((3, 7)), rng.standard_normal(3)
    dy = rng.standard_normal((2, 5, 3))
    xt, wt, bt = (_t(a).requires_grad_(True) for a in (x, w, b))
    (F.linear(xt, wt, bt) * _t(dy)).sum().backward()
    dx, dw, db = dense.linear_bwd(dy, x, w)
    assert rel(dx, xt.grad.numpy()) < 1e-14
    assert rel(dw, wt.grad.numpy()) < 1e-14
    assert rel(db, bt.grad.numpy()) < 1e-14


# ----------------------------------------------------------------- attention
def _sdpa_torch(qkv, n_h, causal):
    nb, ns, e3 = qkv.shape
    e = e3 // 3
    h = e // n_h
    q, k, v = (qkv[..., j * e:(j + 1) * e].reshape(nb, ns, n_h, h).transpose(1, 2) for j in range(3))
    o = F.scaled_dot_product_attention(q, k, v, is_causal=causal)
    return o.transpose(1, 2).reshape(nb, ns, e)


@pytest.mark.parametrize("causal", [True, False])
def test_attention_vs_torch_sdpa(causal):
    rng = np.random.default_rng(7)
    qkv = rng.standard_normal((2, 9, 3 * 12))
    do = rng.standard_normal((2, 9, 12))
    qt = _t(qkv).requires_grad_(True)
    ot = _sdpa_torch(qt, 3, causal)
    (ot * _t(do)).sum().backward()
    o, p = dense.attention_core_fwd(qkv, 3, causal)
    assert rel(o, ot.detach().numpy()) < 1e-13
    dqkv = dense.attention_core_bwd(do, qkv, p, 3)
    assert rel(dqkv, qt.grad.numpy()) < 1e-12


def test_attention_first_query_and_identical_keys():
    rng = np.random.default_rng(8)
    nb, ns, e, nh = 1, 6, 8, 2
    qkv = rng.standard_normal((nb, ns, 3 * e))
    o, p = dense.attention_core_fwd(qkv, nh, True)
    # causal: query 0 sees only key 0 -> P[.,.,0,0] = 1 and O[q=0] = V[0]
    assert np.all(p[:, :, 0, 0] == 1.0)
    assert np.array_equal(o[:, 0], qkv[:, 0, 2 * e:])
    # identical keys -> uniform weights over the causal prefix -> O[q] = mean(V[0..q])
    qkv2 = qkv.copy()
    qkv2[:, :, e:2 * e] = qkv2[:, :1, e:2 * e]
    o2, _ = dense.attention_core_fwd(qkv2, nh, True)
    v = qkv2[0, :, 2 * e:]
    for q in range(ns):
        np.testing.assert_allclose(o2[0, q], v[:q + 1].mean(0), rtol=1e-13, atol=1e-15)


def test_attention_causal_perturbation():
    rng = np.random.default_rng(9)
    qkv = rng.standard_normal((1, 7, 24))
    o, _ = dense.attention_core_fwd(qkv, 2, True)
    qkv2 = qkv.copy()
    qkv2[:, 4:] += rng.standard_normal(qkv2[:, 4:].shape)
    o2, _ = dense.attention_core_fwd(qkv2, 2, True)
    assert np.array_equal(o[:, :4], o2[:, :4])
    assert not np.allclose(o[:, 4:], o2[:, 4:])


def test_attention_softmax_bwd_identity():
    """sum_k P dP = sum_i dO O per query (the D identity used by the kernel)."""
    rng = np.random.default_rng(10)
    nb, ns, e, nh = 2, 8, 12, 3
    qkv = rng.standard_normal((nb, ns, 3 * e))
    do = rng.standard_normal((nb, ns, e))
    o, p = dense.attention_core_fwd(qkv, nh, True)
    q, k, v = dense.split_heads(qkv, nh)
    dob = do.reshape(nb, ns, nh, e // nh).transpose(0, 2, 1, 3)
    ob = o.reshape(nb, ns, nh, e // nh).transpose(0, 2, 1, 3)
    dp = dob @ v.transpose(0, 1, 3, 2)
    np.testing.assert_allclose((p * dp).sum(-1), (dob * ob).sum(-1), rtol=1e-12, atol=1e-14)


# ----------------------------------------------------------------- block
def _torch_block(P, x, n_h, causal):
    e = x.shape[-1]
    h1 = F.layer_norm(x, (e,), P["ln1_g"], P["ln1_b"], 1e-5)
    qkv = F.linear(h1, P["w_qkv"], P["b_qkv"])
    x1 = x + F.linear(_sdpa_torch(qkv, n_h, causal), P["w_o"], P["b_o"])
    h2 = F.layer_norm(x1, (e,), P["ln2_g"], P["ln2_b"], 1e-5)
    g = F.gelu(F.linear(h2, P["w_fc"], P["b_fc"]), approximate="tanh")
    return x1 + F.linear(g, P["w_pr"], P["b_pr"])


@pytest.mark.parametrize("causal", [True, False])
def test_block_vs_torch_autograd(causal):
    E, H, S, B = 16, 2, 6, 2
    params = nnt_inputs.make_params(E, seed=11)
    x = nnt_inputs.make_x(E, S, 0, B, seed=12)
    r = nnt_inputs.make_r(E, S, 0, B, seed=12)
    Pt = {k: _t(v).requires_grad_(True) for k, v in params.items()}
    xt = _t(x).requires_grad_(True)
    yt = _torch_block(Pt, xt, H, causal)
    (yt * _t(r)).sum().backward()
    y, cache = dense.block_fwd(params, x, H, causal)
    assert rel(y, yt.detach().numpy()) < 1e-13
    dx, grads = dense.block_bwd(params, cache, r)
    assert rel(dx, xt.grad.numpy()) < 1e-12
    for k in params:
        assert rel(grads[k], Pt[k].grad.numpy()) < 1e-12, k


def test_block_fd_every_parameter_and_input():
    """Central FD (fp64, h=1e-6) on the micro shape E=8, H=2, S=4, B=2."""
    E, H, S, B = 8, 2, 4, 2
    params = {k: v.astype(np.float64) for k, v in nnt_inputs.make_params(E, seed=21).items()}
    x = nnt_inputs.make_x(E, S, 0, B, seed=22).astype(np.float64)
    r = nnt_inputs.make_r(E, S, 0, B, seed=22).astype(np.float64)

    def loss(P, xx):
        y, _ = dense.block_fwd(P, xx, H, True)
        return float((y * r).sum())

    y, cache = dense.block_fwd(params, x, H, True)
    dx, grads = dense.block_bwd(params, cache, r)
    h = 1e-6
    for name in list(params) + ["x"]:
        base = x if name == "x" else params[name]
        ana = dx if name == "x" else grads[name]
        fd = np.zeros_like(base)
        for idx in np.ndindex(base.shape):
            orig = base[idx]
            base[idx] = orig + h
            lp = loss(params, x)
            base[idx] = orig - h
            lm = loss(params, x)
            base[idx] = orig
            fd[idx] = (lp - lm) / (2 * h)
        assert rel(ana, fd) < 1e-6, name


def test_key_bias_gradient_is_zero():
    """A key bias adds q.b_k to every score of a query row: a per-row constant that the
    softmax (shift-invariant) removes, so dL/db_k = 0 exactly."""
    E, H, S, B = 16, 2, 6, 2
    params = nnt_inputs.make_params(E, seed=13)
    x = nnt_inputs.make_x(E, S, 0, B, seed=14)
    r = nnt_inputs.make_r(E, S, 0, B, seed=14)
    _, cache = dense.block_fwd(params, x, H)
    _, grads = dense.block_bwd(params, cache, r)
    gb = grads["b_qkv"]
    assert np.abs(gb[E:2 * E]).max() < 1e-13 * np.abs(gb).max()
    assert np.abs(gb[:E]).max() > 1e-3 and np.abs(gb[2 * E:]).max() > 1e-3


def test_stack_two_layers_fd_directional():
    E, H, S, B = 8, 2, 4, 2
    layers = [{k: v.astype(np.float64) for k, v in nnt_inputs.make_params(E, seed=31, layer=l).items()}
              for l in range(2)]
    x = nnt_inputs.make_x(E, S, 0, B, seed=32).astype(np.float64)
    r = nnt_inputs.make_r(E, S, 0, B, seed=32).astype(np.float64)
    y, caches = dense.stack_fwd(layers, x, H)
    dx, grads = dense.stack_bwd(layers, caches, r)
    rng = np.random.default_rng(33)
    dirs = [{k: rng.standard_normal(v.shape) for k, v in P.items()} for P in layers]
    dxd = rng.standard_normal(x.shape)
    ana = sum((grads[l][k] * dirs[l][k]).sum() for l in range(2) for k in layers[l]) + (dx * dxd).sum()
    h = 1e-6

    def f(sign):
        Ls = [{k: v + sign * h * dirs[l][k] for k, v in P.items()} for l, P in enumerate(layers)]
        yy, _ = dense.stack_fwd(Ls, x + sign * h * dxd, H)
        return (yy * r).sum()

    fd = (f(1) - f(-1)) / (2 * h)
    assert abs(ana - fd) / abs(fd) < 1e-7


def test_probe_loss_grad():
    rng = np.random.default_rng(34)
    y, r = rng.standard_normal((2, 3, 4)), rng.standard_normal((2, 3, 4))
    T = 6
    h = 1e-6
    g = dense.probe_loss_grad(r, T)
    idx = (1, 2, 3)
    yp, ym = y.copy(), y.copy()
    yp[idx] += h
    ym[idx] -= h
    assert abs((dense.probe_loss(yp, r, T) - dense.probe_loss(ym, r, T)) / (2 * h) - g[idx]) < 1e-8


# ----------------------------------------------------------------- Adam
def test_adam_step1_closed_form():
    rng = np.random.default_rng(40)
    w, g = rng.standard_normal(100), rng.standard_normal(100)
    lr, eps = 1e-3, 1e-8
    w1, m1, v1 = dense.adam_step(w, g, np.zeros(100), np.zeros(100), 1, lr=lr, eps=eps)
    # bias correction makes mhat = g, vhat = g^2 at t = 1
    np.testing.assert_allclose(w1, w - lr * g / (np.abs(g) + eps), rtol=1e-13, atol=1e-16)


def test_adam_zero_grad_and_quadratic():
    w = np.array([0.3, -2.0])
    w1, _, _ = dense.adam_step(w, np.zeros(2), np.zeros(2), np.zeros(2), 1)
    assert np.array_equal(w1, w)
    # f(w) = w^2, w0 = 1, lr = 0.1, 100 steps -> |w| < 0.1
    w, m, v = np.array([1.0]), np.zeros(1), np.zeros(1)
    for t in range(1, 101):
        w, m, v = dense.adam_step(w, 2 * w, m, v, t, lr=0.1)
    assert abs(w[0]) < 0.1


@pytest.mark.parametrize("wd", [0.0, 0.1])
def test_adam_vs_torch_optim(wd):
    rng = np.random.default_rng(41)
    w0 = rng.standard_normal(50)
    grads = [rng.standard_normal(50) for _ in range(5)]
    p = torch.nn.Parameter(_t(w0))
    cls = torch.optim.AdamW if wd else torch.optim.Adam
    opt = cls([p], lr=1e-2, betas=(0.9, 0.999), eps=1e-8, weight_decay=wd)
    w, m, v = w0.copy(), np.zeros(50), np.zeros(50)
    for t, g in enumerate(grads, start=1):
        p.grad = _t(g)
        opt.step()
        w, m, v = dense.adam_step(w, g, m, v, t, lr=1e-2, weight_decay=wd)
    np.testing.assert_allclose(w, p.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_param_count_formula():
    for E in (64, 768, 1600):
        shapes = nnt_inputs.param_shapes(E)
        assert sum(int(np.prod(s)) for s in shapes.values()) == dense.block_param_count(E)


@pytest.mark.parametrize("wd", [0.0, 0.05])
def test_sgd_momentum_vs_torch_optim(wd):
    """SGD with momentum against torch.optim.SGD in fp64 over 4 steps."""
    rng = np.random.default_rng(8)
    w0 = rng.standard_normal(37)
    p = torch.tensor(w0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([p], lr=1e-2, momentum=0.9, weight_decay=wd)
    w, buf = w0.copy(), np.zeros_like(w0)
    for _ in range(4):
        g = rng.standard_normal(37)
        opt.zero_grad()
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        w, buf = dense.sgd_step(w, g, buf, lr=1e-2, momentum=0.9, weight_decay=wd)
        assert np.abs(w - p.detach().numpy()).max() < 1e-15


def test_sgd_zero_momentum_is_plain_gradient_step():
    w, g = np.array([1.0, -2.0]), np.array([0.5, 0.25])
    w1, buf = dense.sgd_step(w, g, np.zeros(2), lr=0.1, momentum=0.0)
    assert np.array_equal(w1, w - 0.1 * g) and np.array_equal(buf, g)
