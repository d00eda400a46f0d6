"""Pins of the GPT-2 shell in oracle/dense.py (embedding layer, tied LM head, cross-entropy;
SURVEY §8(f) f1) against things other than itself: closed forms, torch fp64 library routines
and autograd, the gather/scatter adjoint identity, central finite differences.  No GPU."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import nnt_inputs
from oracle import dense


def _t(a):
    return torch.tensor(np.asarray(a, np.float64), dtype=torch.float64)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_cross_entropy_uniform_logits_is_log_vocab():
    """Equal logits: every class has probability 1/C, so the loss is ln C exactly."""
    for C in (2, 7, 50257):
        x = np.full((3, C), 0.37)
        loss, _ = dense.cross_entropy(x, [0, C // 2, C - 1])
        assert np.allclose(loss, math.log(C), rtol=0, atol=1e-12)


def test_cross_entropy_vs_torch_and_grad():
    rng = np.random.default_rng(3)
    x = 4.0 * rng.standard_normal((9, 31))
    lab = rng.integers(0, 31, 9)
    loss, (m, s) = dense.cross_entropy(x, lab)
    xt = _t(x).requires_grad_(True)
    lt = F.cross_entropy(xt, torch.tensor(lab), reduction="none")
    assert rel(loss, lt.detach().numpy()) < 1e-14
    lt.sum().mul(0.25).backward()
    g = dense.cross_entropy_grad(x, lab, 0.25)
    assert rel(g, xt.grad.numpy()) < 1e-14
    assert np.abs(g.sum(axis=1)).max() < 1e-15          # softmax - onehot: rows sum to zero
    assert np.allclose(m, x.max(axis=1)) and np.allclose(s, np.exp(x - x.max(axis=1, keepdims=True)).sum(1))


def test_cross_entropy_large_logits_no_overflow():
    x = np.array([[1000.0, 0.0, -1000.0]])
    loss, _ = dense.cross_entropy(x, [1])
    assert np.isfinite(loss).all() and abs(loss[0] - 1000.0) < 1e-9


def test_embedding_gather_and_adjoint():
    """embed_bwd is the adjoint of embed_fwd: <fwd(wte, wpe), dx> = <wte, dwte> + <wpe, dwpe>;
    dwte also equals the brute-force scatter-add (np.add.at)."""
    V, S, E, B = 11, 5, 6, 3
    rng = np.random.default_rng(4)
    ids = rng.integers(0, V, (B, S))
    wte, wpe = rng.standard_normal((V, E)), rng.standard_normal((8, E))
    dx = rng.standard_normal((B, S, E))
    x = dense.embed_fwd(ids, wte, wpe)
    assert np.array_equal(x[1, 2], wte[ids[1, 2]] + wpe[2])
    dwte, dwpe = dense.embed_bwd(ids, dx, V, 8)
    lhs = (x * dx).sum()
    rhs = (wte * dwte).sum() + (wpe * dwpe).sum()
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    ref = np.zeros((V, E))
    np.add.at(ref, ids.reshape(-1), dx.reshape(-1, E))
    assert np.allclose(dwte, ref, rtol=0, atol=1e-13)
    assert np.allclose(dwpe[S:], 0) and np.allclose(dwpe[:S], dx.sum(axis=0))


def _model(V, S, E, L, seed=7):
    sh = nnt_inputs.make_shell_params(V, S + 3, E, seed=seed)
    blocks = [nnt_inputs.make_params(E, seed=seed + 1, layer=l, n_layers=L) for l in range(L)]
    return dict(wte=sh["wte"].astype(np.float64), wpe=sh["wpe"].astype(np.float64),
                lnf_g=sh["lnf_g"].astype(np.float64), lnf_b=sh["lnf_b"].astype(np.float64),
                blocks=[{k: v.astype(np.float64) for k, v in b.items()} for b in blocks])


def test_gpt2_vs_torch_autograd():
    """The whole model (embedding, 2 blocks, final LN, tied head, mean CE) against torch fp64
    autograd of the same network built from torch primitives."""
    V, S, E, H, L, B = 37, 6, 16, 2, 2, 2
    model = _model(V, S, E, L)
    tok = nnt_inputs.make_ids(V, S, 0, B, seed=9)
    ids, labels = tok[:, :S], tok[:, 1:]
    loss, cache = dense.gpt2_fwd(model, ids, labels, H)
    g = dense.gpt2_bwd(model, cache)
    from test_oracle_pins import _torch_block
    wte = _t(model["wte"]).requires_grad_(True)
    wpe = _t(model["wpe"]).requires_grad_(True)
    gf, bf = _t(model["lnf_g"]).requires_grad_(True), _t(model["lnf_b"]).requires_grad_(True)
    Pt = [{k: _t(v).requires_grad_(True) for k, v in b.items()} for b in model["blocks"]]
    x = wte[torch.tensor(ids, dtype=torch.long)] + wpe[:S][None]
    for P in Pt:
        x = _torch_block(P, x, H, True)
    hf = F.layer_norm(x, (E,), gf, bf, 1e-5)
    logits = hf.reshape(-1, E) @ wte.T
    lt = F.cross_entropy(logits, torch.tensor(labels.reshape(-1), dtype=torch.long))
    lt.backward()
    assert abs(loss - lt.item()) < 1e-12 * abs(lt.item())
    assert rel(g["wte"], wte.grad.numpy()) < 1e-11
    assert rel(g["wpe"], wpe.grad.numpy()) < 1e-11
    assert rel(g["lnf_g"], gf.grad.numpy()) < 1e-11 and rel(g["lnf_b"], bf.grad.numpy()) < 1e-11
    for l in range(L):
        for k in model["blocks"][l]:
            assert rel(g["blocks"][l][k], Pt[l][k].grad.numpy()) < 1e-11, (l, k)


@pytest.mark.slow
def test_gpt2_fd_shell_parameters():
    """Central FD (h = 1e-6) of the loss w.r.t. every wte / wpe / final-LN entry on a micro model."""
    V, S, E, H, L, B = 7, 4, 8, 2, 1, 2
    model = _model(V, S, E, L, seed=13)
    tok = nnt_inputs.make_ids(V, S, 0, B, seed=14)
    ids, labels = tok[:, :S], tok[:, 1:]
    _, cache = dense.gpt2_fwd(model, ids, labels, H)
    g = dense.gpt2_bwd(model, cache)
    h = 1e-6
    for name in ("wte", "wpe", "lnf_g", "lnf_b"):
        base = model[name]
        fd = np.zeros_like(base)
        for idx in np.ndindex(base.shape):
            o = base[idx]
            base[idx] = o + h
            lp, _ = dense.gpt2_fwd(model, ids, labels, H)
            base[idx] = o - h
            lm, _ = dense.gpt2_fwd(model, ids, labels, H)
            base[idx] = o
            fd[idx] = (lp - lm) / (2 * h)
        assert rel(g[name], fd) < 1e-6, name
