"""GPT-2 shell on the GPU vs the fp64 oracle: the embedding gather/scatter,
the cross-entropy kernel (SoftMax subroutines fused with the loss and its gradient), and the
whole model (embedding, blocks, final LayerNorm, tied LM head, mean cross-entropy, Adam)."""
import numpy as np
import pytest
import torch

import nnt_inputs
from oracle import dense
from gpu_util import close, bf16_round, dev, host, rel

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import model, nnt


def test_embedding_fwd_bit_exact_and_bwd():
    V, S, E, B = 50, 16, 64, 3
    rng = np.random.default_rng(1)
    ids = rng.integers(0, V, (B, S)).astype(np.int32)
    wte = rng.standard_normal((V, E)).astype(np.float32)
    wpe = rng.standard_normal((S + 4, E)).astype(np.float32)
    x = torch.empty(B * S, E, device="cuda")
    I = torch.as_tensor(ids).cuda()
    nnt.nnt_embedding_fwd(I, B * S, S, dev(wte), V, dev(wpe), E, x)
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy().reshape(B, S, E), wte[ids] + wpe[None, :S])
    # integer-valued dx: every sum exact in fp32 -> bit-exact scatter
    dx = rng.integers(-4, 5, (B, S, E)).astype(np.float32)
    dwte = torch.full((V, E), 7.0, device="cuda")
    dwpe = torch.full((S + 4, E), 3.0, device="cuda")
    scr = torch.empty(nnt.nnt_embedding_bwd_scratch_bytes(B * S, V), device="cuda", dtype=torch.uint8)
    # the two accumulate flags act separately (GPT2Model: wte accumulates onto the LM head's
    # half, wpe is overwritten)
    nnt.nnt_embedding_bwd(I, B * S, S, dev(dx), E, dwte, V, dwpe, 1, 0, scr, scr.numel())
    torch.cuda.synchronize()
    want_te, want_pe = dense.embed_bwd(ids, dx, V, S + 4)
    assert np.array_equal(host(dwte), want_te + 7.0)
    assert np.array_equal(host(dwpe)[:S], want_pe[:S])
    assert np.all(host(dwpe)[S:] == 3.0)  # rows >= S untouched
    dwpe.fill_(3.0)
    nnt.nnt_embedding_bwd(I, B * S, S, dev(dx), E, dwte, V, dwpe, 0, 1, scr, scr.numel())
    torch.cuda.synchronize()
    assert np.array_equal(host(dwte), want_te)
    assert np.array_equal(host(dwpe)[:S], want_pe[:S] + 3.0)
    # overwrite mode, real-valued dx
    dx2 = rng.standard_normal((B, S, E)).astype(np.float32)
    dwpe.zero_()
    nnt.nnt_embedding_bwd(I, B * S, S, dev(dx2), E, dwte, V, dwpe, 0, 0, scr, scr.numel())
    torch.cuda.synchronize()
    want_te, want_pe = dense.embed_bwd(ids, dx2, V, S + 4)
    close(host(dwte), want_te, 1e-6, "dwte")
    close(host(dwpe), want_pe, 1e-6, "dwpe")


@pytest.mark.parametrize("T,V", [(2048, 50257), (5000, 300), (9000, 7), (700, 50257), (16384, 50257)])
def test_embedding_bwd_bucket_order(T, V):
    """The scatter sums each id's bucket in ascending token order (the order of the stable counting
    sort; here from a sort of the unique (id, t) keys: chunk bitonic sorts + merge passes, ragged
    last chunk / run for T = 5000 / 9000 / 700): bitwise equal to a sequential fp32 accumulation in
    token order, with heavy repeats (V = 7, 300) and a Zipf-like id mix; and vs the fp64 oracle."""
    S, E = T // 4 if T % 4 == 0 else T, 32
    rng = np.random.default_rng(T + V)
    ids = np.minimum((rng.zipf(1.3, T) - 1), V - 1).astype(np.int32)
    dx = rng.standard_normal((T, E)).astype(np.float32)
    want = np.zeros((V, E), np.float32)
    for t in range(T):  # token order, fp32 adds
        want[ids[t]] += dx[t]
    dwte = torch.full((V, E), 5.0, device="cuda")
    dwpe = torch.zeros((S, E), device="cuda")
    scr = torch.empty(nnt.nnt_embedding_bwd_scratch_bytes(T, V), device="cuda", dtype=torch.uint8)
    I = torch.as_tensor(ids).cuda()
    nnt.nnt_embedding_bwd(I, T, S, dev(dx), E, dwte, V, dwpe, 0, 0, scr, scr.numel())
    torch.cuda.synchronize()
    got = host(dwte)
    assert np.array_equal(got, want), f"max |diff| {np.abs(got - want).max()}"
    if T * V <= 5e7:  # the oracle's one-hot contraction holds T x V doubles
        want64, _ = dense.embed_bwd(ids.reshape(-1, S), dx.reshape(-1, S, E), V, S)
        close(got, want64, 1e-5, "dwte")


@pytest.mark.parametrize("dt", ["f32", "bf16"])
# kernels: bf16 rows <= 104 KB -> persistent double-buffered; rows <= 200 KB -> one staged row per
# CTA (f32 V = 50257, bf16 V = 60001); longer -> the re-reading kernel (f32 V = 60001)
@pytest.mark.parametrize("rows,V", [(37, 1000), (8, 50257), (333, 50257), (301, 4103), (5, 7), (3, 60001)])
def test_cross_entropy_kernel(dt, rows, V):
    rng = np.random.default_rng(2)
    Vp = -(-V // 8) * 8
    x = (3.0 * rng.standard_normal((rows, Vp))).astype(np.float32)
    if dt == "bf16":
        x = bf16_round(x).astype(np.float32)
    lab = rng.integers(0, V, rows).astype(np.int32)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    code = nnt.NNT_BF16 if dt == "bf16" else nnt.NNT_F32
    X = torch.as_tensor(x).cuda().to(tdt)
    L = torch.as_tensor(lab).cuda()
    loss = torch.empty(rows, device="cuda")
    stats = torch.empty(rows, 2, device="cuda")
    D = torch.zeros_like(X)  # padding columns stay defined (host() casts the whole row)
    nnt.nnt_cross_entropy(X, code, rows, V, Vp, L, 0.5, loss, stats, D, Vp)
    torch.cuda.synchronize()
    want, (m, s) = dense.cross_entropy(x[:, :V], lab)
    close(host(loss), want, 1e-5)
    assert np.array_equal(host(stats)[:, 0], m)
    close(host(stats)[:, 1], s, 1e-5, "sumexp")
    g = dense.cross_entropy_grad(x[:, :V], lab, 0.5)
    close(host(D)[:, :V], g, (1e-5 if dt == "f32" else 1e-2))
    # in place over the logits
    nnt.nnt_cross_entropy(X, code, rows, V, Vp, L, 0.5, None, None, X, Vp)
    torch.cuda.synchronize()
    assert torch.equal(X[:, :V], D[:, :V])


def _model_and_oracle(V, E, H, S, B, L, dtype, init, seed=5):
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype=dtype, tile_e=1024 if dtype == "bf16" else 16,
                           tile_f=1024 if dtype == "bf16" else 16, tile_s=1024 if dtype == "bf16" else 16,
                           tile_t=1024 if dtype == "bf16" else 16)
    layers = [nnt_inputs.make_params(E, seed=seed, layer=l, init=init, n_layers=L) for l in range(L)]
    shell = nnt_inputs.make_shell_params(V, S, E, seed=seed + 1, init=init)
    gm = model.GPT2Model(sc, V, layers, shell)
    r = (lambda a: bf16_round(a)) if dtype == "bf16" else (lambda a: np.asarray(a, np.float64))
    om = dict(wte=r(shell["wte"]), wpe=shell["wpe"].astype(np.float64), lnf_g=shell["lnf_g"].astype(np.float64),
              lnf_b=shell["lnf_b"].astype(np.float64),
              blocks=[{k: (r(v) if k.startswith("w_") else v.astype(np.float64)) for k, v in p.items()}
                      for p in layers])
    return gm, om, shell, layers


@pytest.mark.parametrize("cfg", ["f32-tiny", "bf16-small-vocab"])
def test_gpt2_model_vs_oracle(cfg):
    if cfg == "f32-tiny":
        V, E, H, S, B, L, dtype, tol = 128, 64, 2, 32, 2, 2, "f32", 1e-4
    else:
        V, E, H, S, B, L, dtype, tol = 50257, 768, 12, 128, 2, 2, "bf16", 2e-2
    gm, om, shell, layers = _model_and_oracle(V, E, H, S, B, L, dtype, "parity")
    tok = nnt_inputs.make_ids(V, S, 0, B, seed=17)
    ids, labels = tok[:, :S], tok[:, 1:]
    loss = gm.forward(torch.as_tensor(ids).cuda(), torch.as_tensor(labels).cuda()).item()
    gm.backward()
    torch.cuda.synchronize()
    want, cache = dense.gpt2_fwd(om, ids, labels, H)
    g = dense.gpt2_bwd(om, cache)
    assert abs(loss - want) <= tol * abs(want)
    got = {k: host(v) for k, v in gm.grads().items()}
    for k in ("wte", "wpe", "lnf_g", "lnf_b"):
        close(got[k], g[k], tol, k)
    for l in range(L):
        for k, v in gm.stack.grads_of(l).items():
            close(host(v), g["blocks"][l][k], tol, (l, k))


def test_gpt2_graph_equals_eager_bitwise():
    V, E, H, S, B, L = 1000, 768, 12, 128, 2, 2
    outs = []
    for graph in (False, True):
        gm, _, _, _ = _model_and_oracle(V, E, H, S, B, L, "bf16", "gpt2")
        if graph:
            gm.enable_graph()
        losses = []
        for t in range(3):
            tok = torch.as_tensor(nnt_inputs.make_ids(V, S, 0, B, seed=40 + t)).cuda()
            losses.append(gm.train_step(tok[:, :S].contiguous(), tok[:, 1:].contiguous()).item())
        torch.cuda.synchronize()
        outs.append((losses, gm.w.clone(), gm.stack.w.clone(), gm.m.clone()))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1:], outs[1][1:]):
        assert torch.equal(a, b)


def test_gpt2_initial_loss_is_log_vocab():
    """GPT-2 init, real vocabulary: step-0 logits are nearly uniform, loss ~ ln 50257 = 10.825 (+-5%,
    SURVEY f1 pin)."""
    V, E, H, S, B, L = 50257, 768, 12, 128, 2, 2
    gm, _, _, _ = _model_and_oracle(V, E, H, S, B, L, "bf16", "gpt2")
    tok = torch.as_tensor(nnt_inputs.make_ids(V, S, 0, B, seed=3)).cuda()
    loss = gm.forward(tok[:, :S].contiguous(), tok[:, 1:].contiguous()).item()
    assert abs(loss - np.log(V)) < 0.05 * np.log(V)
