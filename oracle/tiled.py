"""The paper's per-tile decomposition, step by step, in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:72 splits data into tiles and operations into per-tile tasks; this
module writes those tasks out literally so that "any tiling gives the untiled
result" (tile-size invariance) can be checked against ``oracle.dense`` and so
that the integer bookkeeping (grids, extents, partitions) has a reference the
C++ host code must match bit for bit.

No blocking, fusion or reordering beyond what the paper's decomposition states.
"""
from __future__ import annotations

import numpy as np

from . import dense

F64 = np.float64


# ---------------------------------------------------------------------------
# Tile bookkeeping
# ---------------------------------------------------------------------------
def tile_grid(shape, tile):
    """grid[d] = ceil(shape[d] / tile[d]); a tile larger than the dim is clamped."""
    if len(shape) != len(tile):
        raise ValueError("rank mismatch")
    out = []
    for s, t in zip(shape, tile):
        if s <= 0 or t <= 0:
            raise ValueError("dims and tiles must be positive")
        t = min(t, s)
        out.append(-(-s // t))
    return out


def tile_extent(dim, tile, idx):
    """Extent of tile ``idx`` along an axis: min(tile, dim - idx*tile) (boundary tiles carry the remainder)."""
    t = min(tile, dim)
    return min(t, dim - idx * t)


def tile_offset(dim, tile, idx):
    return idx * min(tile, dim)


def tile_ranges(dim, tile):
    """[(offset, extent)] for every tile along one axis, in grid order."""
    n = tile_grid([dim], [tile])[0]
    return [(tile_offset(dim, tile, i), tile_extent(dim, tile, i)) for i in range(n)]


def partition(n_units, n_ranks, rank):
    """Units owned by ``rank``: [floor(r n / R), floor((r+1) n / R))."""
    if n_ranks <= 0 or not (0 <= rank < n_ranks) or n_units < 0:
        raise ValueError("bad partition arguments")
    return (rank * n_units) // n_ranks, ((rank + 1) * n_units) // n_ranks


# ---------------------------------------------------------------------------
# Tiled GEMM: C tile (i, j) = sum over K-tiles, ascending
# ---------------------------------------------------------------------------
def gemm_tiled(a, b, tile_m, tile_n, tile_k, alpha=1.0, beta=0.0, c=None):
    """C = alpha * A B + beta * C as a grid of tile products.

    Each output tile accumulates the products of its A row-tiles and B
    column-tiles over the K-tiles in ascending order (the Reduce over the
    contracted tile axis, reading R17: deterministic order).
    """
    a, b = np.asarray(a, F64), np.asarray(b, F64)
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    out = np.zeros((m, n), F64)
    for (i0, ie) in tile_ranges(m, tile_m):
        for (j0, je) in tile_ranges(n, tile_n):
            acc = np.zeros((ie, je), F64)
            for (k0, ke) in tile_ranges(k, tile_k):
                acc = acc + a[i0:i0 + ie, k0:k0 + ke] @ b[k0:k0 + ke, j0:j0 + je]
            out[i0:i0 + ie, j0:j0 + je] = alpha * acc
    if beta != 0.0:
        out = out + beta * np.asarray(c, F64)
    return out


# ---------------------------------------------------------------------------
# SoftMax as two subroutines
# ---------------------------------------------------------------------------
def maxsumexp_tile(t, mask=None):
    """Subroutine 1 on one tile: (t_max, sum e^{t - t_max}) of the tile's entries.

    A fully masked tile returns the merge identity (-inf, 0) (reading R10).
    """
    return dense.maxsumexp(t, mask)


def maxsumexp_merge(m1, s1, m2, s2):
    """(m,s) (+) (m',s') = (M, s e^{m-M} + s' e^{m'-M}), M = max(m, m'); (-inf,0) is the identity."""
    m1, s1, m2, s2 = (np.asarray(z, F64) for z in (m1, s1, m2, s2))
    big = np.maximum(m1, m2)
    safe = np.where(np.isfinite(big), big, 0.0)
    w1 = np.where(np.isfinite(m1), np.exp(m1 - safe), 0.0)
    w2 = np.where(np.isfinite(m2), np.exp(m2 - safe), 0.0)
    return big, s1 * w1 + s2 * w2


def maxsumexp_tiled(t, tile_k, mask=None):
    """Per-tile partials along the last axis merged in ascending tile order."""
    t = np.asarray(t, F64)
    n = t.shape[-1]
    m = np.full(t.shape[:-1], -np.inf)
    s = np.zeros(t.shape[:-1])
    for (k0, ke) in tile_ranges(n, tile_k):
        mk = None if mask is None else mask[..., k0:k0 + ke]
        mj, sj = maxsumexp_tile(t[..., k0:k0 + ke], mk)
        m, s = maxsumexp_merge(m, s, mj, sj)
    return m, s


def softmax_tiled(t, tile_k, mask=None):
    """Subroutine 2: every tile normalised with the aggregated (t_max, denominator)."""
    t = np.asarray(t, F64)
    m, s = maxsumexp_tiled(t, tile_k, mask)
    out = np.zeros_like(t)
    for (k0, ke) in tile_ranges(t.shape[-1], tile_k):
        blk = t[..., k0:k0 + ke]
        val = np.exp(blk - m[..., None]) / s[..., None]
        if mask is not None:
            val = np.where(mask[..., k0:k0 + ke], val, 0.0)
        out[..., k0:k0 + ke] = val
    return out


# ---------------------------------------------------------------------------
# LayerNorm in three steps
# ---------------------------------------------------------------------------
def layernorm_tiled(x, gamma, beta, tile_e, eps=1e-5):
    """Step 1: per E-tile shifted sums S1 = sum(x - c), S2 = sum (x - c)^2 with
    shift c = x[..., 0] (reading R9), accumulated over tiles in ascending order;
    mean = c + S1/E, var = S2/E - (S1/E)^2.  Step 2: normalise every tile.
    Step 3: scale and add bias per tile.  Returns (y, mean, rstd).
    """
    x = np.asarray(x, F64)
    e = x.shape[-1]
    c = x[..., :1]
    s1 = np.zeros(x.shape[:-1])
    s2 = np.zeros(x.shape[:-1])
    for (k0, ke) in tile_ranges(e, tile_e):
        d = x[..., k0:k0 + ke] - c
        s1 = s1 + d.sum(axis=-1)
        s2 = s2 + (d * d).sum(axis=-1)
    mean_shift = s1 / e
    var = np.maximum(s2 / e - mean_shift * mean_shift, 0.0)
    mean = c[..., 0] + mean_shift
    rstd = 1.0 / np.sqrt(var + eps)
    y = np.zeros_like(x)
    for (k0, ke) in tile_ranges(e, tile_e):
        xhat = (x[..., k0:k0 + ke] - mean[..., None]) * rstd[..., None]
        y[..., k0:k0 + ke] = np.asarray(gamma, F64)[k0:k0 + ke] * xhat + np.asarray(beta, F64)[k0:k0 + ke]
    return y, mean, rstd


# ---------------------------------------------------------------------------
# Tiled linear layer and tiled block forward (composition of the above)
# ---------------------------------------------------------------------------
def linear_tiled(x, w, b, tile_t, tile_out, tile_in):
    """Y = W X +. b: tiled GEMM over (tokens, out, in) then per-tile bias add."""
    x2 = np.asarray(x, F64).reshape(-1, x.shape[-1])
    y = gemm_tiled(x2, np.asarray(w, F64).T, tile_t, tile_out, tile_in)
    y = y + np.asarray(b, F64)
    return y.reshape(x.shape[:-1] + (w.shape[0],))


def block_fwd_tiled(params, x, n_h, tiles, causal=True, eps=1e-5):
    """Block forward built only from the tiled subroutines above.

    ``tiles`` = dict(t=token tile, e=embedding tile, f=hidden tile, s=key tile).
    """
    P = {k: np.asarray(v, F64) for k, v in params.items()}
    x = np.asarray(x, F64)
    nb, ns, e = x.shape
    te, tf, tt, ts = tiles["e"], tiles["f"], tiles["t"], tiles["s"]
    h1, _, _ = layernorm_tiled(x, P["ln1_g"], P["ln1_b"], te, eps)
    qkv = linear_tiled(h1, P["w_qkv"], P["b_qkv"], tt, te, te)
    q, k, v = dense.split_heads(qkv, n_h)
    h = q.shape[-1]
    mask = dense.causal_mask(ns) if causal else None
    o = np.zeros_like(q)
    for bi in range(nb):
        for hi in range(n_h):
            a = gemm_tiled(q[bi, hi], k[bi, hi].T, ts, ts, te) / np.sqrt(h)
            p = softmax_tiled(a, ts, mask)
            o[bi, hi] = gemm_tiled(p, v[bi, hi], ts, te, ts)
    om = dense.merge_heads(o)
    x1 = x + linear_tiled(om, P["w_o"], P["b_o"], tt, te, te)
    h2, _, _ = layernorm_tiled(x1, P["ln2_g"], P["ln2_b"], te, eps)
    u = linear_tiled(h2, P["w_fc"], P["b_fc"], tt, tf, te)
    g = dense.gelu(u)  # elementwise: "apply directly to every tile"
    return x1 + linear_tiled(g, P["w_pr"], P["b_pr"], tt, te, tf)
