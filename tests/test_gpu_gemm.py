"""nnt_tile_gemm (SIMT fp32 path and tcgen05 bf16 path) vs the oracle.

Integer-valued inputs in [-4, 4] make every product and fp32 sum exact, so the
tensor-core path must match the oracle BIT-EXACTLY: this pins operand majors
(K-major / MN-major SW128 layouts), transposes, batch strides, ragged M/N/K
tails (TMA zero fill) and causal block skipping.  Real-valued epilogue tests
use the path tolerances.
"""
import math

import numpy as np
import pytest
import torch

import nnt_inputs
from oracle import dense, tiled
from gpu_util import close, bf16_round, dev, host, rel

pytestmark = pytest.mark.gpu

SPLIT_COUNTER_BYTES = 4096 * 4  # the in-kernel split-K reduce's counter zone (gemm_tc.cu kSplitCounters)

if torch.cuda.is_available():
    from paper_2504_13236_b200 import nnt

DT = {"f32": (torch.float32, 0), "bf16": (torch.bfloat16, 1)}


def _op(a, trans):
    return a.T if trans else a


def _run(dtype, ta, tb, M, N, K, a, b, c_dtype="f32", beta=0.0, c0=None, epi=None, alpha=1.0):
    tdt, code = DT[dtype]
    A = dev(a, tdt)
    B = dev(b, tdt)
    ctdt, ccode = DT[c_dtype]
    Cm = dev(c0, ctdt) if c0 is not None else torch.zeros(M, N, device="cuda", dtype=ctdt)
    lda, ldb = a.shape[1], b.shape[1]
    nnt.nnt_tile_gemm(ta, tb, M, N, K, None, alpha, A, code, lda, None, B, code, ldb, None, beta, Cm, ccode, N, None,
                      (1024, 1024, 1024), epi)
    torch.cuda.synchronize()
    return Cm


SHAPES = [(128, 256, 64), (200, 136, 72), (256, 64, 192), (8, 24, 16), (384, 512, 320)]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_integer_bit_exact(dtype, ta, tb, shape):
    M, N, K = shape
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=M + 7 * N + K, kind="int")
    b = nnt_inputs.make_matrix((N, K) if tb else (K, N), seed=3 * M + N + K, kind="int")
    want = tiled.gemm_tiled(_op(a, ta), _op(b, tb), 64, 64, 64)
    got = host(_run(dtype, ta, tb, M, N, K, a, b))
    assert np.array_equal(got, want), f"max |diff| {np.abs(got - want).max()}"


@pytest.mark.parametrize("ta,tb", [(0, 1), (1, 0)])
def test_gemm_bf16_output_rounding_exact(ta, tb):
    M, N, K = 256, 128, 128
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=11, kind="int")
    b = nnt_inputs.make_matrix((N, K) if tb else (K, N), seed=12, kind="int")
    want = bf16_round(tiled.gemm_tiled(_op(a, ta), _op(b, tb), 64, 64, 64))
    got = host(_run("bf16", ta, tb, M, N, K, a, b, c_dtype="bf16"))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("M", [192, 640])  # 640: bf16 runs on CTA pairs (256-row tiles, ragged last pair)
def test_gemm_epilogues(dtype, M):
    N, K = 320, 256
    rng = np.random.default_rng(5)
    a = rng.standard_normal((M, K)).astype(np.float32) / 8
    b = rng.standard_normal((N, K)).astype(np.float32) / 8
    bias = rng.standard_normal(N).astype(np.float32)
    res = rng.standard_normal((M, N)).astype(np.float32)
    c0 = rng.standard_normal((M, N)).astype(np.float32)
    if dtype == "bf16":
        a, b = bf16_round(a), bf16_round(b)
    base = np.asarray(a, np.float64) @ np.asarray(b, np.float64).T
    tol = 1e-5
    # alpha, bias, beta*C, residual (device tensors must outlive the launch: keep references)
    bias_d, res_d = dev(bias), dev(res)
    epi = nnt.make_epilogue(bias=bias_d, residual=res_d, ld_residual=N)
    got = _run(dtype, 0, 1, M, N, K, a, b, beta=0.5, c0=c0, epi=epi, alpha=0.75)
    close(host(got), 0.75 * base + bias + 0.5 * c0 + res, tol)
    # GELU forward: aux <- pre, C <- gelu(pre)
    aux = torch.zeros(M, N, device="cuda", dtype=DT[dtype][0])
    epi = nnt.make_epilogue(bias=bias_d, act=nnt.NNT_ACT_GELU, aux=aux, ld_aux=N)
    got = _run(dtype, 0, 1, M, N, K, a, b, c_dtype=dtype, epi=epi)
    pre = base + bias
    t2 = 1e-6 if dtype == "f32" else 1e-2
    close(host(aux), pre, t2)
    close(host(got), dense.gelu(pre), t2)
    # GELU backward: C <- pre * gelu'(aux)
    u = rng.standard_normal((M, N)).astype(np.float32)
    if dtype == "bf16":
        u = bf16_round(u)
    auxu = dev(u, DT[dtype][0])
    epi = nnt.make_epilogue(act=nnt.NNT_ACT_GELU_BWD, aux=auxu, ld_aux=N)
    got = _run(dtype, 0, 1, M, N, K, a, b, c_dtype=dtype, epi=epi)
    close(host(got), base * dense.gelu_grad(u), t2)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("causal", [0, 1, 2, 3])
def test_gemm_attention_views_and_causal(dtype, causal):
    """Batched (N_b, N_h) views into a fused [B, S, 3E] qkv buffer, integer data."""
    B, S, H, Dh = 2, 384, 3, 64
    E = H * Dh
    tdt, code = DT[dtype]
    qkv = nnt_inputs.make_matrix((B, S, 3 * E), seed=40 + causal, kind="int")
    q = qkv[:, :, :E].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    k = qkv[:, :, E:2 * E].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    Q = dev(qkv, tdt)
    es = Q.element_size()
    sq = (S * 3 * E, Dh)
    batch = (B, H)
    if causal in (0, 1):
        # scores = Q K^T, C [B][H][S][S]
        Cm = torch.zeros(B, H, S, S, device="cuda", dtype=torch.float32)
        epi = nnt.make_epilogue(causal=causal)
        nnt.nnt_tile_gemm(0, 1, S, S, Dh, batch, 1.0, Q, code, 3 * E, sq, Q.data_ptr() + es * E, code, 3 * E, sq, 0.0,
                          Cm, 0, S, (H * S * S, S * S), None, epi)
        torch.cuda.synchronize()
        want = q @ k.transpose(0, 1, 3, 2)
        got = host(Cm)
        if causal:
            mask = np.tril(np.ones((S, S), bool))
            assert np.array_equal(got[..., mask], want[..., mask])
        else:
            assert np.array_equal(got, want)
    else:
        # causal=2: O = P V with P lower triangular; causal=3: dV = P^T dO with P^T upper
        P = nnt_inputs.make_matrix((B, H, S, S), seed=50, kind="int")
        P = P * np.tril(np.ones((S, S), np.float32))
        Pd = dev(P, tdt)
        v = qkv[:, :, 2 * E:].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
        O = torch.zeros(B, S, E, device="cuda", dtype=torch.float32)
        epi = nnt.make_epilogue(causal=causal)
        ta = 0 if causal == 2 else 1
        nnt.nnt_tile_gemm(ta, 0, S, Dh, S, batch, 1.0, Pd, code, S, (H * S * S, S * S), Q.data_ptr() + es * 2 * E,
                          code, 3 * E, sq, 0.0, O, 0, E, (S * E, Dh), None, epi)
        torch.cuda.synchronize()
        Pop = P if causal == 2 else P.transpose(0, 1, 3, 2)
        want = (Pop @ v).transpose(0, 2, 1, 3).reshape(B, S, E)
        assert np.array_equal(host(O), want)


@pytest.fixture(params=["0", "1"], ids=["reduce-kernel", "in-kernel-reduce"])
def splitk_mode(request, monkeypatch):
    """Both split-K reductions: the separate ordered reduce kernel (default) and the in-kernel one
    (NNT_SPLITK_FUSED=1, read by the library at every launch)."""
    monkeypatch.setenv("NNT_SPLITK_FUSED", request.param)
    monkeypatch.setenv("NNT_GEMM_SK", "0")  # split-K itself (stream-K would take these workspaces)
    return request.param


@pytest.mark.parametrize("M,N", [(768, 768), (2304, 768), (768, 3072)])
def test_gemm_split_k_workspace_bit_exact(M, N, splitk_mode):
    """dW-shaped GEMMs (K = T = 8192) split K into a workspace and reduce in split order:
    integer data keeps every partial exact, so the result is bit-exact and run-to-run identical."""
    K = 8192
    a = nnt_inputs.make_matrix((K, M), seed=M + N, kind="int")     # dY  [T][N_out] -> op(A) = dY^T
    b = nnt_inputs.make_matrix((K, N), seed=M * 3 + N, kind="int")  # X   [T][N_in]
    c0 = nnt_inputs.make_matrix((M, N), seed=5, kind="int")
    nb = nnt.nnt_tile_gemm_workspace_bytes(M, N, K, 0)
    assert nb > 0  # the library splits these shapes
    # full size, zero-filled: the in-kernel ordered reduce (arrival counters at the end); run
    # three times -- every launch must leave its counters zero for the next
    ws = torch.zeros(nb, device="cuda", dtype=torch.uint8)
    A, B = dev(a, torch.bfloat16), dev(b, torch.bfloat16)
    want = tiled.gemm_tiled(a.T, b, 256, 256, 1024) + c0
    # the partials alone (no counter space): the separate reduce kernel
    nparts = nb - SPLIT_COUNTER_BYTES
    ws_small = torch.empty(nparts, device="cuda", dtype=torch.uint8)
    for w in (ws, ws_small):
        epi = nnt.make_epilogue(workspace=w)
        for _ in range(3):
            Cm = dev(c0)
            nnt.nnt_tile_gemm(1, 0, M, N, K, None, 1.0, A, 1, M, None, B, 1, N, None, 1.0, Cm, 0, N, None, None, epi)
            torch.cuda.synchronize()
            assert np.array_equal(host(Cm), want)
    assert int(ws[-SPLIT_COUNTER_BYTES:].count_nonzero()) == 0  # counters back to zero


def test_gemm_split_k_shared_workspace_shapes(splitk_mode):
    """The block's four dW GEMMs share one split-K workspace sized for the largest: the in-kernel
    reduce's counter zone (last 16 KB of the workspace) must never lie under another shape's
    partials.  Alternate shapes and K (1024: 2 splits of 8 K-blocks; 8192) on one zero-filled
    workspace, twice round, integer data (exact)."""
    shapes = [(2304, 768), (768, 768), (3072, 768), (768, 3072)]
    Ks = (1024, 8192)
    nb = max(nnt.nnt_tile_gemm_workspace_bytes(M, N, K, 0) for M, N in shapes for K in Ks)
    ws = torch.zeros(nb, device="cuda", dtype=torch.uint8)
    epi = nnt.make_epilogue(workspace=ws)
    for _ in range(2):
        for K in Ks:
            for M, N in shapes:
                a = nnt_inputs.make_matrix((K, M), seed=M + 3 * N + K, kind="int")
                b = nnt_inputs.make_matrix((K, N), seed=M + N + 7 * K, kind="int")
                A, B = dev(a, torch.bfloat16), dev(b, torch.bfloat16)
                Cm = torch.zeros(M, N, device="cuda")
                nnt.nnt_tile_gemm(1, 0, M, N, K, None, 1.0, A, 1, M, None, B, 1, N, None, 0.0, Cm, 0, N, None, None,
                                  epi)
                torch.cuda.synchronize()
                assert np.array_equal(host(Cm), a.T.astype(np.float64) @ b.astype(np.float64)), (M, N, K)
    assert int(ws[-SPLIT_COUNTER_BYTES:].count_nonzero()) == 0


@pytest.mark.parametrize("M,N", [(768, 768), (2304, 768)])
def test_gemm_split_k_real_data_extras(M, N, splitk_mode):
    """Split-K with real-valued data and every extra the ordered reduce applies (alpha, beta*C, bias,
    fp32 residual): in-kernel reduce vs separate reduce kernel vs the fp64 product."""
    K = 8192
    rng = np.random.default_rng(M + N)
    a = bf16_round(rng.standard_normal((K, M)))
    b = bf16_round(rng.standard_normal((K, N)))
    c0 = rng.standard_normal((M, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    res = rng.standard_normal((M, N)).astype(np.float32)
    nb = nnt.nnt_tile_gemm_workspace_bytes(M, N, K, 0)
    nparts = nb - SPLIT_COUNTER_BYTES
    A, B = dev(a, torch.bfloat16), dev(b, torch.bfloat16)
    want = 0.5 * (a.T @ b) + bias + 0.75 * c0 + res
    got = []
    Bias, Res = dev(bias), dev(res)  # alive until the launches have run
    for w in (torch.zeros(nb, device="cuda", dtype=torch.uint8), torch.empty(nparts, device="cuda", dtype=torch.uint8)):
        epi = nnt.make_epilogue(workspace=w, bias=Bias, residual=Res, ld_residual=N)
        Cm = dev(c0)
        nnt.nnt_tile_gemm(1, 0, M, N, K, None, 0.5, A, 1, M, None, B, 1, N, None, 0.75, Cm, 0, N, None, None, epi)
        torch.cuda.synchronize()
        got.append(host(Cm))
        close(got[-1], want, 1e-5)
    close(got[0], got[1], 1e-6)


# Stream-K shapes: (M, N, K, ta, tb, residual) -- the GPT-2 XL projections the schedule takes
# (long K, >= 2 whole data-parallel waves, a last wave <= 82 % full): 8192 x 1600 with K = 6400 /
# 4800 (224 pair tiles on 74 pairs: 2 data-parallel waves + 76 tiles over 74 units), the dW-shaped
# 1600 x 6400 x 8192 (175 tiles, beta = 2 here), and a ragged M / N residual GEMM.
SK_SHAPES = [(8192, 1600, 6400, 0, 1, False), (8192, 1600, 4800, 0, 0, False), (1600, 6400, 8192, 1, 0, False),
             (8000, 1560, 6400, 0, 1, True)]


@pytest.mark.parametrize("shape", SK_SHAPES, ids=lambda s: "x".join(map(str, s[:3])) + ("r" if s[5] else ""))
def test_gemm_stream_k_bit_exact(shape, capfd, monkeypatch):
    """Stream-K schedule (the last wave's K-block iterations spread over all units; a tile shared by
    several units finished by the one holding its last K-block, which adds the others' fp32
    partials): integer data keeps every partial exact, so C must equal the exact product with beta*C,
    bias and residual; three launches on one zero-filled workspace (the flags must come back to 0)."""
    monkeypatch.setenv("NNT_DEBUG_GEMM", "1")
    monkeypatch.setenv("NNT_GEMM_SK", "1")  # opt-in schedule
    M, N, K, ta, tb, with_res = shape
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=M + N + K, kind="int")
    b = nnt_inputs.make_matrix((N, K) if tb else (K, N), seed=3 * M + N + 5 * K, kind="int")
    c0 = nnt_inputs.make_matrix((M, N), seed=9, kind="int")
    bias = nnt_inputs.make_matrix((1, N), seed=10, kind="int")[0]
    res = nnt_inputs.make_matrix((M, N), seed=11, kind="int")
    nb = nnt.nnt_tile_gemm_workspace_bytes(M, N, K, 0)
    ws = torch.zeros(nb, device="cuda", dtype=torch.uint8)
    A, B = dev(a, torch.bfloat16), dev(b, torch.bfloat16)
    Bias, Res = dev(bias), dev(res)
    epi = (nnt.make_epilogue(workspace=ws, bias=Bias, residual=Res, ld_residual=N) if with_res
           else nnt.make_epilogue(workspace=ws, bias=Bias))
    want = _op(a, ta).astype(np.float64) @ _op(b, tb).astype(np.float64) + bias + 2.0 * c0 + (res if with_res else 0)
    lda, ldb = a.shape[1], b.shape[1]
    for _ in range(3):
        Cm = dev(c0)
        nnt.nnt_tile_gemm(ta, tb, M, N, K, None, 1.0, A, 1, lda, None, B, 1, ldb, None, 2.0, Cm, 0, N, None, None, epi)
        torch.cuda.synchronize()
        got = host(Cm)
        assert np.array_equal(got, want), f"max |diff| {np.abs(got - want).max()}"
    assert "stream-K" in capfd.readouterr().err  # the schedule really ran
    assert int(ws[-SPLIT_COUNTER_BYTES:].count_nonzero()) == 0  # flags consumed


@pytest.mark.parametrize("act", ["gelu", "gelu_bwd", "plain"])
def test_gemm_stream_k_bf16_epilogues_vs_data_parallel(act, monkeypatch):
    """bf16-output stream-K GEMMs with the fused epilogues (bias + GELU storing the pre-activation,
    GELU' with the aux input) on real data: against the fp64 product (bf16 tolerance) and against
    the data-parallel schedule (NNT_GEMM_SK=0; only the K association of the shared tiles differs),
    and bitwise reproducible run to run."""
    M, N, K = 8192, 1600, 6400
    rng = np.random.default_rng(17)
    a = bf16_round(rng.standard_normal((M, K)) / 16)
    b = bf16_round(rng.standard_normal((N, K)) / 16)
    bias = rng.standard_normal(N).astype(np.float32) / 4
    u = bf16_round(rng.standard_normal((M, N)))
    A, B, Bias, U = dev(a, torch.bfloat16), dev(b, torch.bfloat16), dev(bias), dev(u, torch.bfloat16)
    monkeypatch.setenv("NNT_GEMM_SK", "1")  # (the workspace size includes the stream-K slots)
    ws = torch.zeros(nnt.nnt_tile_gemm_workspace_bytes(M, N, K, 1, 1), device="cuda", dtype=torch.uint8)
    base = a.astype(np.float64) @ b.astype(np.float64).T
    outs = []
    for sk in ("1", "1", "0"):
        monkeypatch.setenv("NNT_GEMM_SK", sk)
        Cm = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        aux = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        if act == "gelu":
            epi = nnt.make_epilogue(workspace=ws, bias=Bias, act=nnt.NNT_ACT_GELU, aux=aux, ld_aux=N)
        elif act == "gelu_bwd":
            epi = nnt.make_epilogue(workspace=ws, act=nnt.NNT_ACT_GELU_BWD, aux=U, ld_aux=N)
        else:
            epi = nnt.make_epilogue(workspace=ws)
        nnt.nnt_tile_gemm(0, 1, M, N, K, None, 1.0, A, 1, K, None, B, 1, K, None, 0.0, Cm, 1, N, None, None, epi)
        torch.cuda.synchronize()
        outs.append((host(Cm), host(aux)))
    if act == "gelu":
        close(outs[0][1], base + bias, 1e-2)
        close(outs[0][0], dense.gelu(base + bias), 1e-2)
    elif act == "gelu_bwd":
        close(outs[0][0], base * dense.gelu_grad(u), 1e-2)
    else:
        close(outs[0][0], base, 1e-2)
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])  # reproducible
    close(outs[0][0], outs[2][0], 1e-2)  # vs the data-parallel schedule
    assert int(ws[-SPLIT_COUNTER_BYTES:].count_nonzero()) == 0


@pytest.mark.parametrize("ta,tb", [(0, 1), (1, 0), (0, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(512, 384, 256), (296, 200, 136), (1000, 520, 72), (2048, 2304, 128)])
def test_gemm_cta_pair_bit_exact(ta, tb, shape):
    """Unbatched non-causal bf16 GEMMs with M >= 256 run on CTA pairs (tcgen05 cta_group::2, M=256
    MMAs, each CTA staging half of the B tile): both operand majors, ragged M/N/K tails (a pair whose
    second CTA lies wholly past M), BN = 128 and 256 pair tiles."""
    M, N, K = shape
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=M + N + 1, kind="int")
    b = nnt_inputs.make_matrix((N, K) if tb else (K, N), seed=M + 2 * N, kind="int")
    want = tiled.gemm_tiled(_op(a, ta), _op(b, tb), 64, 64, 64)
    got = host(_run("bf16", ta, tb, M, N, K, a, b))
    assert np.array_equal(got, want), f"max |diff| {np.abs(got - want).max()}"
    gotb = host(_run("bf16", ta, tb, M, N, K, a, b, c_dtype="bf16"))
    assert np.array_equal(gotb, bf16_round(want))


@pytest.mark.parametrize("M,N,K,ta", [(768, 768, 8192, 1), (3072, 768, 8192, 1), (768, 3072, 8192, 1),
                                       (296, 200, 136, 1), (200, 136, 72, 1), (512, 384, 256, 0)])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_gemm_a_rowsum_bias_grad_bit_exact(M, N, K, ta, beta):
    """R27: a_rowsum = beta * a_rowsum + sum_k op(A)[i][k] fused into the GEMM (tensor cores against
    a ones vector) -- the bias gradient of a dW = dY^T X GEMM.  Integer data: C and the row sums
    are exact; covers single-CTA and CTA-pair tiles, split-K (workspace) and unsplit GEMMs."""
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=M + K, kind="int")
    b = nnt_inputs.make_matrix((K, N), seed=N + K, kind="int")
    c0 = nnt_inputs.make_matrix((M, N), seed=7, kind="int")
    r0 = nnt_inputs.make_matrix((M,), seed=8, kind="int")
    nb = nnt.nnt_tile_gemm_workspace_bytes(M, N, K, 0)
    ws = torch.zeros(max(nb, 16), device="cuda", dtype=torch.uint8)
    rs = dev(r0)
    epi = nnt.make_epilogue(workspace=ws if nb else None, a_rowsum=rs)
    A, B, Cm = dev(a, torch.bfloat16), dev(b, torch.bfloat16), dev(c0)
    nnt.nnt_tile_gemm(ta, 0, M, N, K, None, 1.0, A, 1, a.shape[1], None, B, 1, N, None, beta, Cm, 0, N, None, None, epi)
    torch.cuda.synchronize()
    opa = (a.T if ta else a).astype(np.float64)
    assert np.array_equal(host(Cm), opa @ b.astype(np.float64) + beta * c0)
    assert np.array_equal(host(rs), opa.sum(axis=1) + beta * r0)


@pytest.mark.parametrize("N", [768, 3072])
def test_gemm_wave_model_tile_widths_bit_exact(N):
    """M = 8192 rows with N = 768 / 3072: wave-model tile widths on CTA pairs."""
    M, K = 8192, 256
    a = nnt_inputs.make_matrix((M, K), seed=N, kind="int")
    b = nnt_inputs.make_matrix((N, K), seed=N + 1, kind="int")
    got = host(_run("bf16", 0, 1, M, N, K, a, b))
    assert np.array_equal(got, a.astype(np.float64) @ b.T.astype(np.float64))


@pytest.mark.parametrize("causal", [0, 1])
def test_scores_gemm_fused_maxsumexp_partials(causal):
    """Softmax subroutine 1 per 32-key tile in the score-GEMM epilogue + nnt_maxsumexp_merge
    equals the oracle's (max, sumexp) of the same scores."""
    B, S, H, Dh = 2, 384, 3, 64
    E = H * Dh
    rng = np.random.default_rng(61 + causal)
    qkv = bf16_round(rng.standard_normal((B, S, 3 * E)))
    Q = dev(qkv, torch.bfloat16)
    sq = (S * 3 * E, Dh)
    alpha = 1.0 / math.sqrt(Dh)
    scores = torch.zeros(B, H, S, S, device="cuda")
    nparts = S // 32
    part = torch.zeros(B * H * S, nparts, 2, device="cuda")
    epi = nnt.make_epilogue(causal=causal, row_stats=part, ld_row_stats=nparts)
    nnt.nnt_tile_gemm(0, 1, S, S, Dh, (B, H), alpha, Q, 1, 3 * E, sq, Q.data_ptr() + 2 * E, 1, 3 * E, sq, 0.0, scores,
                      0, S, (H * S * S, S * S), None, epi)
    stats = torch.zeros(B * H * S, 2, device="cuda")
    nnt.nnt_maxsumexp_merge(part, B * H * S, nparts, nparts, 32, causal, S, stats)
    torch.cuda.synchronize()
    q = qkv[:, :, :E].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    k = qkv[:, :, E:2 * E].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    a = alpha * (q @ k.transpose(0, 1, 3, 2))
    mask = np.tril(np.ones((S, S), bool)) if causal else None
    m_ref, s_ref = dense.maxsumexp(a, mask)
    got = host(stats).reshape(B, H, S, 2)
    np.testing.assert_allclose(got[..., 0], m_ref, rtol=1e-5, atol=1e-5)
    close(got[..., 1], s_ref, 1e-5)


@pytest.mark.parametrize("causal", [0, 1])
@pytest.mark.parametrize("S", [384, 200])
def test_rowstats_then_softmax_gemms(causal, S):
    """R26: the statistics pass (NNT_ACT_ROWSTATS: subroutine 1 aggregated over all key tiles of
    a row on chip, no scores stored) and the P pass (NNT_ACT_SOFTMAX: subroutine 2 on the
    recomputed score tile) vs the oracle's maxsumexp / softmax of the same scores."""
    B, H, Dh = 2, 3, 64
    E = H * Dh
    rng = np.random.default_rng(81 + causal + S)
    qkv = bf16_round(2.0 * rng.standard_normal((B, S, 3 * E)))
    Q = dev(qkv, torch.bfloat16)
    sq = (S * 3 * E, Dh)
    alpha = 1.0 / math.sqrt(Dh)
    stats = torch.full((B * H * S, 2), float("nan"), device="cuda")
    epi = nnt.make_epilogue(act=nnt.NNT_ACT_ROWSTATS, causal=causal, row_stats=stats)
    nnt.nnt_tile_gemm(0, 1, S, S, Dh, (B, H), alpha, Q, 1, 3 * E, sq, Q.data_ptr() + 2 * E, 1, 3 * E, sq, 0.0, None,
                      0, S, (H * S * S, S * S), None, epi)
    P = torch.full((B, H, S, S), float("nan"), device="cuda", dtype=torch.bfloat16)
    epi2 = nnt.make_epilogue(act=nnt.NNT_ACT_SOFTMAX, causal=causal, row_stats=stats)
    nnt.nnt_tile_gemm(0, 1, S, S, Dh, (B, H), alpha, Q, 1, 3 * E, sq, Q.data_ptr() + 2 * E, 1, 3 * E, sq, 0.0, P,
                      1, S, (H * S * S, S * S), None, epi2)
    torch.cuda.synchronize()
    q = qkv[:, :, :E].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    k = qkv[:, :, E:2 * E].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    a = alpha * (q @ k.transpose(0, 1, 3, 2))
    mask = np.tril(np.ones((S, S), bool)) if causal else None
    m_ref, s_ref = dense.maxsumexp(a, mask)
    got = host(stats).reshape(B, H, S, 2)
    np.testing.assert_allclose(got[..., 0], m_ref, rtol=1e-5, atol=1e-5)
    close(got[..., 1], s_ref, 1e-5)
    p = host(P)
    p_ref = dense.softmax(a, mask)
    r, c = np.arange(S)[:, None], np.arange(S)[None, :]
    written = c < np.minimum(S, (r // 128 + 1) * 128) if causal else np.ones((S, S), bool)
    assert not np.isnan(p[..., written]).any() and np.isnan(p[..., ~written]).all()
    if causal:
        assert np.all(p[..., written & (c > r)] == 0.0)
    close(np.where(written, p, 0.0), p_ref, 4e-3)  # bf16 rounding of P
    np.testing.assert_allclose(np.where(written, p, 0.0).sum(-1), 1.0, atol=2e-2)


def test_fused_softmax_bwd_gemm_and_rowdot():
    """dA = P * (dO V^T - D) / sqrt(h) from the dP GEMM epilogue, with D = rowdot(dO, O)
    (identity sum_k P dP = sum_i dO O), vs the oracle's softmax backward (R18)."""
    B, S, H, Dh = 2, 384, 3, 64
    E = H * Dh
    rng = np.random.default_rng(71)
    qkv = bf16_round(rng.standard_normal((B, S, 3 * E)))
    do = bf16_round(rng.standard_normal((B, S, E)))
    o_ref, p_ref = dense.attention_core_fwd(qkv, H, True)
    P16 = bf16_round(p_ref)
    O16 = bf16_round(o_ref)
    Qd, dOd = dev(qkv, torch.bfloat16), dev(do, torch.bfloat16)
    Pd, Od = dev(P16, torch.bfloat16), dev(O16, torch.bfloat16)
    D = torch.zeros(B * H * S, device="cuda")
    nnt.nnt_attn_rowdot(dOd, Od, 1, B, S, H, Dh, D)
    dA = torch.full((B, H, S, S), float("nan"), device="cuda", dtype=torch.bfloat16)
    scale = 1.0 / math.sqrt(Dh)
    epi = nnt.make_epilogue(act=nnt.NNT_ACT_SOFTMAX_BWD, aux=Pd, ld_aux=S, causal=1, rowvec=D, rowscale=scale)
    nnt.nnt_tile_gemm(0, 1, S, S, Dh, (B, H), 1.0, dOd, 1, E, (S * E, Dh), Qd.data_ptr() + 2 * 2 * E, 1, 3 * E,
                      (S * 3 * E, Dh), 0.0, dA, 1, S, (H * S * S, S * S), None, epi)
    torch.cuda.synchronize()
    dob = do.reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    ob = O16.reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    close(host(D).reshape(B, H, S), (dob * ob).sum(-1), 1e-5)
    v = qkv[:, :, 2 * E:].reshape(B, S, H, Dh).transpose(0, 2, 1, 3)
    want = scale * dense.softmax_bwd(P16, dob @ v.transpose(0, 1, 3, 2))
    got = host(dA)
    mask = np.tril(np.ones((S, S), bool))
    assert np.all(got[..., ~mask & (np.arange(S)[None, :] < ((np.arange(S)[:, None] // 128 + 1) * 128))] == 0.0)
    close(np.where(mask, got, 0.0), want, 2e-2)


@pytest.mark.parametrize("dt,h", [("bf16", 64), ("bf16", 8), ("bf16", 16), ("bf16", 256), ("bf16", 24),
                                  ("f32", 64), ("f32", 12), ("f32", 128)])
def test_attn_rowdot_head_dims(dt, h):
    """D[b, n, s] = sum_i dO[b, s, n, i] O[b, s, n, i] (R18's row-dot identity) for head dims that
    take the lane-cooperative kernel (h x 2 B / 16 a power of two) and the thread-per-row one."""
    B, S, H = 2, 77, 5
    rng = np.random.default_rng(72 + h)
    do = bf16_round(rng.standard_normal((B, S, H, h)))
    o = bf16_round(rng.standard_normal((B, S, H, h)))
    tdt, code = DT[dt]
    D = torch.full((B * H * S,), float("nan"), device="cuda")
    nnt.nnt_attn_rowdot(dev(do, tdt), dev(o, tdt), code, B, S, H, h, D)
    torch.cuda.synchronize()
    want = (do * o).sum(-1).transpose(0, 2, 1)  # [B, H, S]
    close(host(D).reshape(B, H, S), want, 1e-6)


def test_gemm_rejects_bad_arguments():
    A = torch.zeros(64, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(nnt.NNTError) as e:  # misaligned leading dimension for TMA
        nnt.nnt_tile_gemm(0, 1, 64, 64, 60, None, 1.0, A, 1, 60, None, A, 1, 60, None, 0.0, A, 1, 64, None)
    assert e.value.status == nnt.NNT_ERR_ALIGN
    with pytest.raises(nnt.NNTError) as e:  # mixed operand dtypes
        nnt.nnt_tile_gemm(0, 1, 64, 64, 64, None, 1.0, A, 1, 64, None, A, 0, 64, None, 0.0, A, 1, 64, None)
    assert e.value.status == nnt.NNT_ERR_DTYPE


# Narrow tail tiles: (M, N, K, ta, tb) with N % BN != 0 -- the GPT-2 XL N = 1600 shapes (7th pair
# tile column 64 wide), a remainder that is not a multiple of 32 (1616: 80 -> 96 / 128-wide MMAs), a
# split-K dW shape (1600 x 1600 x 8192, MN-major operands), single-CTA tiles (M < 256)
TAIL_SHAPES = [(8192, 1600, 1600, 0, 1), (8192, 1600, 640, 0, 0), (1024, 1616, 256, 1, 0), (640, 1560, 192, 1, 1),
               (1600, 1600, 8192, 1, 0), (200, 1600, 128, 0, 1)]


@pytest.mark.parametrize("shape", TAIL_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_gemm_narrow_tail_bit_exact(shape, capfd, monkeypatch):
    """The last N column of tiles runs N = tail_n MMAs (the remainder rounded up to 32; a CTA pair
    stages tail_n / 2 B rows per CTA) and, M-outer, after every full tile: on integer data C must
    equal the exact product plus bias and 2*C0 (fp32 out) / its bf16 rounding (bf16 out), exactly
    as with full-width tail MMAs (NNT_GEMM_TAIL=0)."""
    monkeypatch.setenv("NNT_DEBUG_GEMM", "1")
    M, N, K, ta, tb = shape
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=M + N + K, kind="int")
    b = nnt_inputs.make_matrix((N, K) if tb else (K, N), seed=3 * M + N + 5 * K, kind="int")
    c0 = nnt_inputs.make_matrix((M, N), seed=9, kind="int")
    bias = nnt_inputs.make_matrix((1, N), seed=10, kind="int")[0]
    ws = torch.zeros(nnt.nnt_tile_gemm_workspace_bytes(M, N, K, 0), device="cuda", dtype=torch.uint8)
    A, B, Bias = dev(a, torch.bfloat16), dev(b, torch.bfloat16), dev(bias)
    want = _op(a, ta).astype(np.float64) @ _op(b, tb).astype(np.float64)
    lda, ldb = a.shape[1], b.shape[1]
    for tail in ("1", "0"):
        monkeypatch.setenv("NNT_GEMM_TAIL", tail)
        Cm = dev(c0)
        epi = nnt.make_epilogue(workspace=ws, bias=Bias)
        nnt.nnt_tile_gemm(ta, tb, M, N, K, None, 1.0, A, 1, lda, None, B, 1, ldb, None, 2.0, Cm, 0, N, None, None, epi)
        Cb = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        nnt.nnt_tile_gemm(ta, tb, M, N, K, None, 1.0, A, 1, lda, None, B, 1, ldb, None, 0.0, Cb, 1, N, None, None,
                          nnt.make_epilogue(workspace=ws))
        torch.cuda.synchronize()
        got = host(Cm)
        assert np.array_equal(got, want + bias + 2.0 * c0), f"tail={tail} max |diff| {np.abs(got - want).max()}"
        assert np.array_equal(host(Cb), bf16_round(want)), f"tail={tail} bf16"
        err = capfd.readouterr().err
        launches = [l for l in err.splitlines() if l.startswith("gemm_tc launch")]
        assert launches, err
        import re
        for l in launches:
            bn, cg = int(re.search(r" BN (\d+)", l).group(1)), int(re.search(r" CG (\d+)", l).group(1))
            gran = 32 if tb else 64 * cg  # MN-major B: 64-element halves per CTA
            tn = -(-(N % bn) // gran) * gran
            if tail == "1" and N % bn and tn < bn:
                assert f" tail {tn}" in l, l  # the narrow MMAs really ran
            else:
                assert " tail 0" in l, l


@pytest.mark.parametrize("ta,tb", [(1, 0), (0, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(1600, 1600, 1024), (512, 1536, 320), (8192, 1600, 192)])
def test_gemm_blocked_mn_major_maps_bit_exact(ta, tb, shape, monkeypatch):
    """MN-major operands with MN % 64 == 0 are staged by ONE 5-D TMA request per stage (dims {64, K,
    MN / 64, ...}; all the stage's 64-element blocks) instead of one request per block: on integer
    data the product is exact either way (NNT_GEMM_BLOCKED=0 restores the 4-D maps), with the M / N
    tails past the last whole block zero-filled by the block dimension's bound."""
    M, N, K = shape
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=M + 7 * N + K, kind="int")
    b = nnt_inputs.make_matrix((N, K) if tb else (K, N), seed=5 * M + N + 3 * K, kind="int")
    want = _op(a, ta).astype(np.float64) @ _op(b, tb).astype(np.float64)
    for blk in ("1", "0"):
        monkeypatch.setenv("NNT_GEMM_BLOCKED", blk)
        got = host(_run("bf16", ta, tb, M, N, K, a, b))
        assert np.array_equal(got, want), f"blocked={blk} max |diff| {np.abs(got - want).max()}"
        gotb = host(_run("bf16", ta, tb, M, N, K, a, b, c_dtype="bf16"))
        assert np.array_equal(gotb, bf16_round(want)), f"blocked={blk} bf16"


@pytest.mark.parametrize("shape", [(8192, 768, 3072), (2048, 576, 320)], ids=lambda s: "x".join(map(str, s)))
def test_gemm_pair192_exception_bit_exact(shape, capfd, monkeypatch):
    """K-major-B GEMMs whose 256-wide CTA-pair tiles fill under 70 % of their rounds (GPT-2 small's
    N = 768 projection: 96 tiles on 74 pairs) run on 192-wide pair tiles (96 B rows per CTA): on
    integer data with bias, 2*C0 and an fp32 residual the product is exact with the exception on and
    off (NNT_GEMM_192_EXC=0: 256-wide tiles)."""
    monkeypatch.setenv("NNT_DEBUG_GEMM", "1")
    M, N, K = shape
    a = nnt_inputs.make_matrix((M, K), seed=M + N + 2 * K, kind="int")
    b = nnt_inputs.make_matrix((N, K), seed=7 * M + N + K, kind="int")
    c0 = nnt_inputs.make_matrix((M, N), seed=19, kind="int")
    bias = nnt_inputs.make_matrix((1, N), seed=20, kind="int")[0]
    res = nnt_inputs.make_matrix((M, N), seed=21, kind="int")
    A, B, Bias, Res = dev(a, torch.bfloat16), dev(b, torch.bfloat16), dev(bias), dev(res)
    want = a.astype(np.float64) @ b.astype(np.float64).T + bias + 2.0 * c0 + res
    import re
    seen = {}
    for exc in ("1", "0"):
        monkeypatch.setenv("NNT_GEMM_192_EXC", exc)
        Cm = dev(c0)
        epi = nnt.make_epilogue(bias=Bias, residual=Res, ld_residual=N)
        nnt.nnt_tile_gemm(0, 1, M, N, K, None, 1.0, A, 1, K, None, B, 1, K, None, 2.0, Cm, 0, N, None, None, epi)
        torch.cuda.synchronize()
        got = host(Cm)
        assert np.array_equal(got, want), f"exc={exc} max |diff| {np.abs(got - want).max()}"
        launches = [l for l in capfd.readouterr().err.splitlines() if l.startswith("gemm_tc launch")]
        seen[exc] = [(int(re.search(r" BN (\d+)", l).group(1)), int(re.search(r" CG (\d+)", l).group(1)))
                     for l in launches]
    if M == 8192:  # the GPT-2 small projection shape takes the exception
        assert seen["1"] == [(192, 2)] and seen["0"] != [(192, 2)], seen


@pytest.mark.parametrize("shape", [(8192, 1600, 1600), (8192, 768, 3072), (1000, 1560, 256), (640, 320, 2048)],
                         ids=lambda s: "x".join(map(str, s)))
def test_gemm_residual_tma_staged_bit_exact(shape, monkeypatch):
    """The fp32 residual of the out-projection / projection epilogues TMA-staged chunk by chunk through
    the epilogue warps' staging buffers (IN_RES_SMEM: 3-4 chunks per warp and tile over 2 buffers,
    each refilled once its chunk's store has read it): on integer data with bias, 2*C0 and the
    residual, C is exact with the staged path and with the register prefetch (NNT_GEMM_RES_SMEM=0),
    for CTA-pair and single-CTA tiles and ragged M / N edges."""
    M, N, K = shape
    a = nnt_inputs.make_matrix((M, K), seed=3 * M + N + K, kind="int")
    b = nnt_inputs.make_matrix((N, K), seed=M + 5 * N + K, kind="int")
    c0 = nnt_inputs.make_matrix((M, N), seed=29, kind="int")
    bias = nnt_inputs.make_matrix((1, N), seed=30, kind="int")[0]
    res = nnt_inputs.make_matrix((M, N), seed=31, kind="int")
    A, B, Bias, Res = dev(a, torch.bfloat16), dev(b, torch.bfloat16), dev(bias), dev(res)
    want = a.astype(np.float64) @ b.astype(np.float64).T + bias + 2.0 * c0 + res
    for rs in ("1", "0"):
        monkeypatch.setenv("NNT_GEMM_RES_SMEM", rs)
        for _ in range(2):
            Cm = dev(c0)
            epi = nnt.make_epilogue(bias=Bias, residual=Res, ld_residual=N)
            nnt.nnt_tile_gemm(0, 1, M, N, K, None, 1.0, A, 1, K, None, B, 1, K, None, 2.0, Cm, 0, N, None, None, epi)
            torch.cuda.synchronize()
            got = host(Cm)
            assert np.array_equal(got, want), f"res_smem={rs} max |diff| {np.abs(got - want).max()}"
