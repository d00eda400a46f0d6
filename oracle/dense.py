"""Plain, untiled fp64 definitions of the GPT-2 block forward/backward and Adam.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the
product path.

Layout: activations are NumPy arrays ``[N_b, N_s, N_e]`` (row-major, embedding
fastest), which is the paper's ``N_e x N_s x N_b`` tensor with its first index
fastest.  Q/K/V for head ``n`` occupy columns
``n*h .. n*h+h-1`` of the q/k/v thirds of the fused QKV projection
(reading R5/R6 in DESIGN.md).

Everything here is the textbook definition; a library primitive (``@``,
``np.exp``, ``np.max``) may serve as a step, nothing is blocked or fused.
"""
from __future__ import annotations

import math

import numpy as np

F64 = np.float64

# GELU tanh-approximation constants (reading R11: GPT-2 "gelu_new").
GELU_C = math.sqrt(2.0 / math.pi)
GELU_A = 0.044715


def _f64(a):
    return np.asarray(a, dtype=F64)


# ---------------------------------------------------------------------------
# Elementwise: nonlinear activation
# ---------------------------------------------------------------------------
def gelu(u):
    """gelu(u) = 0.5 u (1 + tanh(c (u + a u^3))), c = sqrt(2/pi), a = 0.044715.

    PAPER.md:142-145 ("nonlinear activations ... elementwise"); the concrete
    function is reading R11 (GPT-2 tanh approximation).
    """
    u = _f64(u)
    return 0.5 * u * (1.0 + np.tanh(GELU_C * (u + GELU_A * u ** 3)))


def gelu_grad(u):
    """d gelu / du = 0.5 (1 + t) + 0.5 u (1 - t^2) c (1 + 3 a u^2), t = tanh(c(u + a u^3))."""
    u = _f64(u)
    t = np.tanh(GELU_C * (u + GELU_A * u ** 3))
    return 0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * GELU_C * (1.0 + 3.0 * GELU_A * u * u)


def gelu_bwd(u, dy):
    """du = dy * gelu'(u) (chain rule, reading R18)."""
    return _f64(dy) * gelu_grad(u)


# ---------------------------------------------------------------------------
# Linear layer Y = W X +. b
# ---------------------------------------------------------------------------
def linear_fwd(x, w, b):
    """Y = W X +. b with X rows = tokens: y[t, d] = sum_e w[d, e] x[t, e] + b[d].

    PAPER.md:152: W is N_d x N_e, the bias is added over the unchanged
    dimensions (N_s, N_b).
    """
    x, w, b = _f64(x), _f64(w), _f64(b)
    return x @ w.T + b


def linear_bwd(dy, x, w):
    """dX = dY W,  dW = dY^T X,  db = sum_t dY  (reading R18)."""
    dy, x, w = _f64(dy), _f64(x), _f64(w)
    d_out = dy.shape[-1]
    d_in = x.shape[-1]
    dy2 = dy.reshape(-1, d_out)
    x2 = x.reshape(-1, d_in)
    dx = (dy2 @ w).reshape(x.shape)
    dw = dy2.T @ x2
    db = dy2.sum(axis=0)
    return dx, dw, db


# ---------------------------------------------------------------------------
# LayerNorm
# ---------------------------------------------------------------------------
def layernorm_fwd(x, gamma, beta, eps=1e-5):
    """y = gamma * (x - mu) / sqrt(var + eps) + beta over the embedding axis.

    PAPER.md:162: "mean and variance of every tile accumulation, normalization
    of every tile and scaling with an addition of bias".  Untiled here: the
    statistics are the plain mean and the biased (1/N_e) variance (reading R9).
    Returns (y, mean, rstd) with rstd = 1/sqrt(var + eps).
    """
    x, gamma, beta = _f64(x), _f64(gamma), _f64(beta)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mu) * rstd
    return gamma * xhat + beta, mu[..., 0], rstd[..., 0]


def layernorm_bwd(dy, x, gamma, mean, rstd):
    """Textbook LayerNorm gradient (reading R18).

    dxhat = dy * gamma
    dx    = rstd * (dxhat - mean_e(dxhat) - xhat * mean_e(dxhat * xhat))
    dgamma = sum_t dy * xhat,  dbeta = sum_t dy
    """
    dy, x, gamma = _f64(dy), _f64(x), _f64(gamma)
    mean, rstd = _f64(mean)[..., None], _f64(rstd)[..., None]
    xhat = (x - mean) * rstd
    dxhat = dy * gamma
    dx = rstd * (dxhat - dxhat.mean(axis=-1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(axis=-1, keepdims=True))
    e = x.shape[-1]
    dgamma = (dy * xhat).reshape(-1, e).sum(axis=0)
    dbeta = dy.reshape(-1, e).sum(axis=0)
    return dx, dgamma, dbeta


# ---------------------------------------------------------------------------
# SoftMax
# ---------------------------------------------------------------------------
def maxsumexp(t, mask=None):
    """The two quantities the paper's first softmax subroutine produces.

    t_max = max_i t_i and denominator sum_k e^{t_k - t_max} over the last
    axis.  ``mask`` (bool, True = keep) excludes entries;
    an all-masked slice yields (-inf, 0) (reading R10).
    """
    t = _f64(t)
    if mask is not None:
        t = np.where(mask, t, -np.inf)
    m = t.max(axis=-1)
    safe = np.where(np.isfinite(m), m, 0.0)
    s = np.exp(t - safe[..., None]).sum(axis=-1)
    return m, s


def softmax(t, mask=None):
    """p_i = e^{t_i - t_max} / sum_k e^{t_k - t_max}, masked -> 0."""
    t = _f64(t)
    if mask is not None:
        t = np.where(mask, t, -np.inf)
    m = t.max(axis=-1, keepdims=True)
    e = np.exp(t - m)
    return e / e.sum(axis=-1, keepdims=True)


def softmax_bwd(p, dp):
    """dA = P * (dP - sum_k P dP)  (Jacobian of softmax applied to dP, reading R18)."""
    p, dp = _f64(p), _f64(dp)
    return p * (dp - (p * dp).sum(axis=-1, keepdims=True))


# ---------------------------------------------------------------------------
# Attention
# ---------------------------------------------------------------------------
def causal_mask(n_s):
    """mask[q, k] = (k <= q): GPT-2 autoregressive mask (reading R2)."""
    return np.tril(np.ones((n_s, n_s), dtype=bool))


def split_heads(qkv, n_h):
    """qkv [N_b, N_s, 3 N_e] -> q, k, v each [N_b, N_h, N_s, h] (reading R5/R6)."""
    nb, ns, e3 = qkv.shape
    e = e3 // 3
    h = e // n_h
    parts = []
    for j in range(3):
        blk = qkv[:, :, j * e:(j + 1) * e].reshape(nb, ns, n_h, h)
        parts.append(blk.transpose(0, 2, 1, 3))
    return parts


def merge_heads(o):
    """[N_b, N_h, N_s, h] -> [N_b, N_s, N_h*h] with column n*h + i (reading R5)."""
    nb, nh, ns, h = o.shape
    return o.transpose(0, 2, 1, 3).reshape(nb, ns, nh * h)


def attention_core_fwd(qkv, n_h, causal=True):
    """B = V SoftMax(K^T Q / sqrt(h)) per (batch, head).

    With row-major [query, key] scores A[q,k] = sum_i Q[q,i] K[k,i] / sqrt(h)
    (the paper's K^T Q, keys first; softmax over keys, reading R3), P =
    softmax_k(A), O[q,i] = sum_k P[q,k] V[k,i].  Returns (O merged [N_b,N_s,N_e],
    P [N_b,N_h,N_s,N_s]).
    """
    qkv = _f64(qkv)
    q, k, v = split_heads(qkv, n_h)
    h = q.shape[-1]
    a = (q @ k.transpose(0, 1, 3, 2)) / math.sqrt(h)
    mask = causal_mask(a.shape[-1]) if causal else None
    p = softmax(a, mask)
    o = p @ v
    return merge_heads(o), p


def attention_core_bwd(do_merged, qkv, p, n_h):
    """Gradients of attention_core_fwd w.r.t. qkv (reading R18).

    dP = dO V^T, dV = P^T dO, dA = P*(dP - sum_k P dP), dQ = dA K / sqrt(h),
    dK = dA^T Q / sqrt(h).
    """
    qkv, p = _f64(qkv), _f64(p)
    q, k, v = split_heads(qkv, n_h)
    h = q.shape[-1]
    nb, ns, e = do_merged.shape
    do = _f64(do_merged).reshape(nb, ns, n_h, h).transpose(0, 2, 1, 3)
    dp = do @ v.transpose(0, 1, 3, 2)
    dv = p.transpose(0, 1, 3, 2) @ do
    da = softmax_bwd(p, dp)
    dq = (da @ k) / math.sqrt(h)
    dk = (da.transpose(0, 1, 3, 2) @ q) / math.sqrt(h)
    return np.concatenate([merge_heads(dq), merge_heads(dk), merge_heads(dv)], axis=-1)


# ---------------------------------------------------------------------------
# GPT-2 block (pre-LN wiring, reading R1)
# ---------------------------------------------------------------------------
PARAM_NAMES = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
               "ln2_g", "ln2_b", "w_fc", "b_fc", "w_pr", "b_pr")


def block_fwd(params, x, n_h, causal=True, eps=1e-5):
    """One GPT-2 block forward.

      h1 = LN(x; g1, b1)
      qkv = h1 W_qkv^T + b_qkv
      O  = attention(qkv)
      x1 = x + O W_o^T + b_o                   PAPER.md:181 ("Y = W B^T"), residual R1
      h2 = LN(x1; g2, b2)
      u  = h2 W_fc^T + b_fc ; g = gelu(u)
      y  = x1 + g W_pr^T + b_pr
    Returns (y, cache) where cache holds what block_bwd needs.
    """
    P = {k: _f64(v) for k, v in params.items()}
    x = _f64(x)
    h1, mu1, r1 = layernorm_fwd(x, P["ln1_g"], P["ln1_b"], eps)
    qkv = linear_fwd(h1, P["w_qkv"], P["b_qkv"])
    o, p = attention_core_fwd(qkv, n_h, causal)
    x1 = x + linear_fwd(o, P["w_o"], P["b_o"])
    h2, mu2, r2 = layernorm_fwd(x1, P["ln2_g"], P["ln2_b"], eps)
    u = linear_fwd(h2, P["w_fc"], P["b_fc"])
    g = gelu(u)
    y = x1 + linear_fwd(g, P["w_pr"], P["b_pr"])
    cache = dict(x=x, h1=h1, mu1=mu1, r1=r1, qkv=qkv, p=p, o=o, x1=x1,
                 h2=h2, mu2=mu2, r2=r2, u=u, g=g, n_h=n_h)
    return y, cache


def block_bwd(params, cache, dy):
    """Backward of block_fwd (chain rule; reading R18).  Returns (dx, grads)."""
    P = {k: _f64(v) for k, v in params.items()}
    c = cache
    dy = _f64(dy)
    grads = {}
    # y = x1 + g W_pr^T + b_pr
    dg, grads["w_pr"], grads["b_pr"] = linear_bwd(dy, c["g"], P["w_pr"])
    du = gelu_bwd(c["u"], dg)
    dh2, grads["w_fc"], grads["b_fc"] = linear_bwd(du, c["h2"], P["w_fc"])
    dx1_ln, grads["ln2_g"], grads["ln2_b"] = layernorm_bwd(dh2, c["x1"], P["ln2_g"], c["mu2"], c["r2"])
    dx1 = dy + dx1_ln
    # x1 = x + O W_o^T + b_o
    do, grads["w_o"], grads["b_o"] = linear_bwd(dx1, c["o"], P["w_o"])
    dqkv = attention_core_bwd(do, c["qkv"], c["p"], c["n_h"])
    dh1, grads["w_qkv"], grads["b_qkv"] = linear_bwd(dqkv, c["h1"], P["w_qkv"])
    dx_ln, grads["ln1_g"], grads["ln1_b"] = layernorm_bwd(dh1, c["x"], P["ln1_g"], c["mu1"], c["r1"])
    dx = dx1 + dx_ln
    return dx, grads


def stack_fwd(layers, x, n_h, causal=True, eps=1e-5):
    """L blocks applied in order; returns (y, caches)."""
    caches = []
    for params in layers:
        x, cache = block_fwd(params, x, n_h, causal, eps)
        caches.append(cache)
    return x, caches


def stack_bwd(layers, caches, dy):
    """Backward through the stack, last layer first; returns (dx, [grads per layer])."""
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        dy, grads[l] = block_bwd(layers[l], caches[l], dy)
    return dy, grads


# ---------------------------------------------------------------------------
# Block-only loss (reading R13): linear probe L = (1/T_global) sum_t <y_t, r_t>
# ---------------------------------------------------------------------------
def probe_loss(y, r, t_global):
    return float((_f64(y) * _f64(r)).sum() / t_global)


def probe_loss_grad(r, t_global):
    """dL/dy = r / T_global (independent of y)."""
    return _f64(r) / t_global


# ---------------------------------------------------------------------------
# GPT-2 shell: embedding layer, tied LM head, cross-entropy
# ---------------------------------------------------------------------------
def embed_fwd(ids, wte, wpe):
    """x[b, s] = wte[ids[b, s]] + wpe[s].

    PAPER.md:133-137 (the embedding layer equips every token with an N_e vector from an
    N_v x N_e table); the learned position table wpe is GPT-2's (reading R29)."""
    ids = np.asarray(ids)
    return _f64(wte)[ids] + _f64(wpe)[None, : ids.shape[1], :]


def embed_bwd(ids, dx, n_vocab, n_pos):
    """dwte[v] = sum_{(b,s): ids[b,s] = v} dx[b, s];  dwpe[s] = sum_b dx[b, s].

    Written as the one-hot contraction dwte = onehot(ids)^T dx (the adjoint of the gather)."""
    ids = np.asarray(ids).reshape(-1)
    dx = _f64(dx)
    onehot = np.zeros((ids.size, n_vocab))
    onehot[np.arange(ids.size), ids] = 1.0
    dwte = onehot.T @ dx.reshape(-1, dx.shape[-1])
    dwpe = np.zeros((n_pos, dx.shape[-1]))
    dwpe[: dx.shape[1]] = dx.sum(axis=0)
    return dwte, dwpe


def cross_entropy(logits, labels):
    """Per-sample loss  -log( e^{x_c} / sum_j e^{x_j} )  (sign typo read as the
    positive NLL, reading R13), computed through the SoftMax subroutines:
    (M, S) = maxsumexp(x) per row, loss = log S + M - x_c.  Returns (per-row loss, stats)."""
    x = _f64(logits)
    m, ssum = maxsumexp(x)                 # per row: (max, sumexp) = softmax subroutine 1
    rows = np.arange(x.shape[0])
    loss = np.log(ssum) + m - x[rows, np.asarray(labels)]
    return loss, (m, ssum)


def cross_entropy_grad(logits, labels, scale):
    """d(scale * sum_rows loss)/dx = scale * (softmax(x) - onehot(c))."""
    p = softmax(_f64(logits))
    p[np.arange(p.shape[0]), np.asarray(labels)] -= 1.0
    return scale * p


def gpt2_fwd(model, ids, labels, n_h, causal=True, eps=1e-5):
    """Full GPT-2: embedding -> L pre-LN blocks -> final LayerNorm -> tied LM head -> mean CE.

    model: dict with 'wte' [V, E], 'wpe' [S_max, E], 'lnf_g', 'lnf_b' [E] and 'blocks' (list of
    block parameter dicts).  Loss = (1/T) sum_t CE_t (mean over tokens, reading R13).
    Returns (loss, cache)."""
    x0 = embed_fwd(ids, model["wte"], model["wpe"])
    xl, caches = stack_fwd(model["blocks"], x0, n_h, causal, eps)
    hf, mu, r = layernorm_fwd(xl, model["lnf_g"], model["lnf_b"], eps)
    b, s, e = hf.shape
    logits = hf.reshape(-1, e) @ _f64(model["wte"]).T
    loss_rows, _ = cross_entropy(logits, np.asarray(labels).reshape(-1))
    t = b * s
    cache = dict(ids=np.asarray(ids), labels=np.asarray(labels).reshape(-1), caches=caches, xl=xl, hf=hf, mu=mu,
                 r=r, logits=logits, t=t)
    return float(loss_rows.sum() / t), cache


def gpt2_bwd(model, cache, t_global=None):
    """Gradients of gpt2_fwd's loss (scaled by 1/t_global; default the batch's T) w.r.t. every
    parameter: dict with 'wte' (LM head + embedding, tied), 'wpe', 'lnf_g', 'lnf_b', 'blocks'."""
    t_global = cache["t"] if t_global is None else t_global
    wte = _f64(model["wte"])
    dlogits = cross_entropy_grad(cache["logits"], cache["labels"], 1.0 / t_global)
    hf = cache["hf"]
    b, s, e = hf.shape
    dhf = (dlogits @ wte).reshape(b, s, e)
    dwte = dlogits.T @ hf.reshape(-1, e)
    dxl, dlnf_g, dlnf_b = layernorm_bwd(dhf, cache["xl"], model["lnf_g"], cache["mu"], cache["r"])
    dx0, gblocks = stack_bwd(model["blocks"], cache["caches"], dxl)
    dwte_e, dwpe = embed_bwd(cache["ids"], dx0, wte.shape[0], _f64(model["wpe"]).shape[0])
    return dict(wte=dwte + dwte_e, wpe=dwpe, lnf_g=dlnf_g, lnf_b=dlnf_b, blocks=gblocks)


# ---------------------------------------------------------------------------
# Adam / AdamW (reading R12)
# ---------------------------------------------------------------------------
def adam_step(w, g, m, v, t, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8,
              weight_decay=0.0):
    """One Kingma-Ba Adam step with bias correction; t is the 1-based step.

    m <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2
    w <- w - lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)  [- lr*wd*w for AdamW]
    Returns new (w, m, v).
    """
    w, g, m, v = _f64(w), _f64(g), _f64(m), _f64(v)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** t)
    vhat = v / (1.0 - beta2 ** t)
    w_new = w - lr * mhat / (np.sqrt(vhat) + eps)
    if weight_decay:
        w_new = w_new - lr * weight_decay * w
    return w_new, m, v


def sgd_step(w, g, buf, lr=1e-2, momentum=0.9, weight_decay=0.0):
    """SGD with momentum ("a weighted sum of the input vector, gradient, and
    momentum term"), the usual heavy-ball form: buf <- momentum * buf + (g + wd * w);
    w <- w - lr * buf.  buf starts at 0 (so the first step's buf is the gradient).
    Returns new (w, buf)."""
    w, g, buf = _f64(w), _f64(g), _f64(buf)
    d = g + weight_decay * w if weight_decay else g
    buf = momentum * buf + d
    return w - lr * buf, buf


# ---------------------------------------------------------------------------
# Work counts used for reporting
# ---------------------------------------------------------------------------
def block_param_count(e):
    """12 E^2 + 13 E parameters per block (4 linears + 2 LayerNorms)."""
    return 12 * e * e + 13 * e
