"""The fused attention tile kernels (R33) against the fp64 oracle, through the C-ABI.

nnt_attention_fwd_pv: softmax subroutine 2 from the row statistics (the ROWSTATS score GEMM, R26)
and O = P V, P staged once; nnt_attention_bwd_kv: dA = P (dP - D) / sqrt(h) written over the P tile
in shared memory and stored (query-major), dK = dA^T Q and dV = P^T dO accumulated on chip; dQ = dA K
by nnt_tile_gemm on the stored dA.
Shapes span several 128-row tiles (S = 256, 384), causal and not, B * H > 1; bf16 tolerance 2e-2
norm-wise and element-wise (gpu_util.close).  The block tests (test_gpu_block / test_gpu_shapes /
test_gpu_parity_full) run the same kernels inside nnt_block_fwd / _bwd.
"""
import math

import numpy as np
import pytest
import torch

from oracle import dense
from gpu_util import bf16_round, close, dev, host

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import nnt

H_D = 64


def _inputs(B, S, H, seed):
    rng = np.random.default_rng(seed)
    E = H * H_D
    qkv = bf16_round(rng.standard_normal((B, S, 3 * E)) * 1.5)  # peaked, non-trivial softmax rows
    do = bf16_round(rng.standard_normal((B, S, E)))
    return qkv, do


def _rowstats(Q, B, S, H, scale, causal):
    """Softmax subroutine 1 by the library's ROWSTATS score GEMM (as nnt_block_fwd runs it)."""
    E = H * H_D
    stats = torch.empty(B * H * S, 2, device="cuda")
    q = Q.reshape(-1).view(torch.uint8)  # byte offsets: K starts 2 * E bytes into a row
    sq = [S * 3 * E, H_D]
    epi = nnt.make_epilogue(act=nnt.NNT_ACT_ROWSTATS, row_stats=stats,
                            causal=nnt.NNT_CAUSAL_OUT_LOWER if causal else nnt.NNT_CAUSAL_NONE)
    nnt.nnt_tile_gemm(0, 1, S, S, H_D, [B, H], scale, q, 1, 3 * E, sq, q[2 * E:], 1, 3 * E, sq, 0.0, None, 0, S,
                      [H * S * S, S * S], None, epi)
    return stats


@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("B,S,H", [(2, 256, 3), (1, 384, 2), (2, 1024, 4)])
def test_attention_stats_kernel(B, S, H, causal):
    """nnt_attention_stats (softmax subroutine 1 on recomputed score tiles, R26) vs the oracle's
    maxsumexp of the scaled scores, and vs the ROWSTATS score GEMM (both up to fp32 rounding)."""
    E = H * H_D
    scale = 1.0 / np.sqrt(H_D)
    qkv, _ = _inputs(B, S, H, seed=S + H + 7 * causal)
    Q = dev(qkv, torch.bfloat16)
    st = torch.full((B * H * S, 2), float("nan"), device="cuda")
    nnt.nnt_attention_stats(Q, B, S, H, H_D, scale, causal, st)
    ref_gemm = _rowstats(Q, B, S, H, scale, causal)
    torch.cuda.synchronize()
    q_, k_, _ = dense.split_heads(qkv, H)
    x = (q_ @ k_.transpose(0, 1, 3, 2)) * scale
    if causal:
        x = np.where(dense.causal_mask(S), x, -np.inf)
    want_m, want_s = dense.maxsumexp(x.reshape(-1, S))  # (max, sumexp) per row
    got = host(st)
    close(got[:, 0], want_m, 1e-5, "max")
    close(got[:, 1], want_s, 1e-5, "sumexp")
    close(got, host(ref_gemm), 1e-5, "vs ROWSTATS GEMM")


def _written(S, causal):
    """Mask of the 128 x 128 (query, key) tiles the kernels write: all, or kb <= qb."""
    t = np.arange(S) // 128
    return (t[None, :] <= t[:, None]) if causal else np.ones((S, S), bool)


@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("B,S,H", [(2, 256, 3), (1, 384, 2)])
def test_fused_attention_fwd_bwd(B, S, H, causal):
    assert nnt.nnt_attention_fused_supported(S, H_D)
    E = H * H_D
    scale = 1.0 / math.sqrt(H_D)
    qkv, do = _inputs(B, S, H, seed=S + H + causal)
    Q = dev(qkv, torch.bfloat16)
    stats = _rowstats(Q, B, S, H, scale, causal)
    P = torch.full((B, H, S, S), float("nan"), device="cuda", dtype=torch.bfloat16)
    O = torch.empty(B, S, E, device="cuda", dtype=torch.bfloat16)
    nnt.nnt_attention_fwd_pv(Q, B, S, H, H_D, scale, causal, stats, P, O)
    torch.cuda.synchronize()
    o_ref, p_ref = dense.attention_core_fwd(qkv, H, causal=bool(causal))
    w = _written(S, causal)
    p = host(P)
    assert np.all(np.isfinite(p[:, :, w]))
    close(p[:, :, w], p_ref[:, :, w], 2e-2, "P")
    if causal:  # masked entries of the written diagonal tiles are exactly zero
        m = w & ~dense.causal_mask(S)
        assert np.all(p[:, :, m] == 0.0)
    close(host(O), o_ref, 2e-2, "O")

    # backward: D = rowdot(dO, O), then the fused dA / dK / dV pass and the dQ GEMM
    dO = dev(do, torch.bfloat16)
    D = torch.empty(B * H * S, device="cuda")
    nnt.nnt_attn_rowdot(dO, O, nnt.NNT_BF16, B, S, H, H_D, D)
    dA = torch.full((B, H, S, S), float("nan"), device="cuda", dtype=torch.bfloat16)
    dqkv = torch.zeros(B, S, 3 * E, device="cuda", dtype=torch.bfloat16)
    nnt.nnt_attention_bwd_kv(Q, dO, P, D, B, S, H, H_D, scale, causal, dA, dqkv)
    sp = [H * S * S, S * S]
    sq = [S * 3 * E, H_D]
    qb = Q.reshape(-1).view(torch.uint8)
    epi = nnt.make_epilogue(causal=nnt.NNT_CAUSAL_A_LOWER if causal else nnt.NNT_CAUSAL_NONE)
    nnt.nnt_tile_gemm(0, 0, S, H_D, S, [B, H], 1.0, dA, 1, S, sp, qb[2 * E:], 1, 3 * E, sq, 0.0, dqkv, 1, 3 * E,
                      sq, None, epi)
    torch.cuda.synchronize()
    # oracle backward from the P the GPU produced (isolates the backward kernels)
    p_used = np.where(w, p, 0.0)
    want = dense.attention_core_bwd(do, qkv, p_used, H)
    got = host(dqkv)
    for j, name in enumerate(("dQ", "dK", "dV")):
        close(got[..., j * E:(j + 1) * E], want[..., j * E:(j + 1) * E], 2e-2, name)
    # dA (query-major) on the written tiles: the oracle's dA / sqrt(h)
    q_, k_, v_ = dense.split_heads(qkv, H)
    do_h = do.reshape(B, S, H, H_D).transpose(0, 2, 1, 3)
    da_ref = dense.softmax_bwd(p_used, do_h @ v_.transpose(0, 1, 3, 2)) * scale
    da = host(dA)
    close(da[:, :, w], da_ref[:, :, w], 2e-2, "dA")


def test_fused_attention_rejects_unsupported():
    assert not nnt.nnt_attention_fused_supported(192, 64)
    assert not nnt.nnt_attention_fused_supported(256, 32)
    x = torch.zeros(16, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(nnt.NNTError):
        nnt.nnt_attention_fwd_pv(x, 1, 192, 1, 64, 0.125, 1, x, x, x)
