"""Tile-size invariance of the oracle: the paper's per-tile decomposition
(oracle/tiled.py) equals the untiled definition (oracle/dense.py) for any
tiling, including non-divisible boundary tiles; plus the bit-exact integer
bookkeeping examples from SPEC S:247-251."""
import numpy as np
import pytest

import nnt_inputs
from oracle import dense, tiled


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_tile_grid_examples():
    assert tiled.tile_grid([4, 4], [2, 2]) == [2, 2]
    assert tiled.tile_grid([5, 3], [2, 3]) == [3, 1]
    assert tiled.tile_extent(5, 2, 2) == 1
    assert tiled.tile_grid([768], [1024]) == [1]          # clamped
    assert [e for _, e in tiled.tile_ranges(2304, 1024)] == [1024, 1024, 256]
    assert [e for _, e in tiled.tile_ranges(4800, 1024)] == [1024] * 4 + [704]
    assert [e for _, e in tiled.tile_ranges(6400, 1024)] == [1024] * 6 + [256]
    with pytest.raises(ValueError):
        tiled.tile_grid([0], [4])
    with pytest.raises(ValueError):
        tiled.tile_grid([4], [0])


def test_tile_ranges_cover_exactly():
    rng = np.random.default_rng(0)
    for _ in range(200):
        d, t = int(rng.integers(1, 300)), int(rng.integers(1, 400))
        rs = tiled.tile_ranges(d, t)
        assert rs[0][0] == 0
        assert sum(e for _, e in rs) == d
        for (o1, e1), (o2, _) in zip(rs, rs[1:]):
            assert o1 + e1 == o2


def test_partition_covers_and_balances():
    for n in range(0, 40):
        for R in range(1, 9):
            parts = [tiled.partition(n, R, r) for r in range(R)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("seed", range(8))
def test_gemm_tiled_equals_dense(seed):
    rng = np.random.default_rng(seed)
    m, n, k = (int(v) for v in rng.integers(1, 70, 3))
    a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
    tm, tn, tk = (int(v) for v in rng.integers(1, 40, 3))
    assert rel(tiled.gemm_tiled(a, b, tm, tn, tk), a @ b) < 1e-13


@pytest.mark.parametrize("seed", range(8))
def test_softmax_tiled_equals_dense(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 90))
    t = 20 * rng.standard_normal((5, n))
    tile = int(rng.integers(1, 100))
    mask = np.tril(np.ones((5, n), bool), k=int(rng.integers(0, n)))
    m1, s1 = tiled.maxsumexp_tiled(t, tile, mask)
    m0, s0 = dense.maxsumexp(t, mask)
    assert np.array_equal(m1, m0)          # max is exact under any split
    assert rel(s1, s0) < 1e-13
    assert rel(tiled.softmax_tiled(t, tile, mask), dense.softmax(t, mask)) < 1e-13


def test_maxsumexp_merge_identity_and_fully_masked_tile():
    m, s = tiled.maxsumexp_merge(-np.inf, 0.0, 2.0, 3.0)
    assert m == 2.0 and s == 3.0
    m, s = tiled.maxsumexp_merge(-np.inf, 0.0, -np.inf, 0.0)
    assert m == -np.inf and s == 0.0 and np.isfinite(s)
    t = np.array([[1.0, 2.0, 5.0, 7.0]])
    mask = np.array([[True, True, False, False]])
    m, s = tiled.maxsumexp_tiled(t, 2, mask)   # second tile fully masked
    assert m[0] == 2.0 and abs(s[0] - (1 + np.exp(-1))) < 1e-15


@pytest.mark.parametrize("seed", range(8))
def test_layernorm_tiled_equals_dense(seed):
    rng = np.random.default_rng(200 + seed)
    e = int(rng.integers(2, 130))
    x = 100.0 + 3 * rng.standard_normal((4, e))     # |mean| >> std: shifted sums matter
    g, b = rng.standard_normal(e), rng.standard_normal(e)
    tile = int(rng.integers(1, 150))
    y1, m1, r1 = tiled.layernorm_tiled(x, g, b, tile)
    y0, m0, r0 = dense.layernorm_fwd(x, g, b)
    assert rel(y1, y0) < 1e-11
    assert rel(m1, m0) < 1e-14


@pytest.mark.parametrize("tiles", [dict(t=16, e=16, f=16, s=16), dict(t=24, e=24, f=24, s=24),
                                   dict(t=7, e=5, f=33, s=9), dict(t=4096, e=4096, f=4096, s=4096)])
def test_block_fwd_tiled_equals_dense(tiles):
    cfg = nnt_inputs.CONFIGS["tiny"]
    params = nnt_inputs.make_params(cfg.E, seed=1234)
    x = nnt_inputs.make_x(cfg.E, cfg.S, 0, cfg.B, seed=5678)
    y0, _ = dense.block_fwd(params, x, cfg.H)
    y1 = tiled.block_fwd_tiled(params, x, cfg.H, tiles)
    assert rel(y1, y0) < 1e-12
