"""bf16 tensor-core path at the other BASELINE.json shapes, and the bench configuration itself.

* One block of the GPT-2 large (E=1280, H=20), XL (E=1600, H=25: boundary tiles 1024+576,
  4800 = 4x1024+704, 6400 = 6x1024+256) and wide (E=8192, H=128) shapes vs the fp64 oracle,
  every tensor rel <= 2e-2 (north_star's bf16 tolerance).
* The exact configuration bench.py times (GPT-2 small, 12 layers, B=8, S=1024, GPT-2 init,
  one CUDA-graph training step): y and dx of sampled sequences vs the oracle run on those
  sequences alone (every block is independent across sequences: LayerNorm is per token,
  attention per (sequence, head), the probe-loss gradient dy = r / T per token).
"""
import numpy as np
import pytest
import torch

import nnt_inputs
from oracle import dense
from gpu_util import close, bf16_round, dev, host, rel

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import model


def _used(p):
    """The parameters the GPU computes with: bf16-rounded weight matrices, fp32 vectors."""
    return {k: (bf16_round(v) if k.startswith("w_") else v.astype(np.float64)) for k, v in p.items()}


@pytest.mark.timeout(600)
@pytest.mark.parametrize("E,H,S,B", [(1280, 20, 1024, 1), (1600, 25, 1024, 1), (8192, 128, 128, 1)],
                         ids=["large", "xl", "wide"])
def test_bf16_block_baseline_shapes(E, H, S, B):
    sc = model.StackConfig(L=1, E=E, H=H, S=S, B=B, dtype="bf16")
    layers = [nnt_inputs.make_params(E, seed=4321, init="parity")]
    st = model.BlockStack(sc, layers)
    x = nnt_inputs.make_x(E, S, 0, B, seed=21)
    r = nnt_inputs.make_r(E, S, 0, B, seed=21)
    st.forward(dev(x))
    st.probe_loss(dev(r))
    dx_dev = st.backward()
    torch.cuda.synchronize()
    used = _used(layers[0])
    del layers
    y_ref, cache = dense.block_fwd(used, x, H)
    dx_ref, g_ref = dense.block_bwd(used, cache, dense.probe_loss_grad(r, B * S))
    close(host(st.xs[-1]), y_ref, 2e-2)
    close(host(dx_dev), dx_ref, 2e-2)
    for n, gv in st.grads_of(0).items():
        close(host(gv), g_ref[n], 2e-2, n)


@pytest.mark.timeout(900)
def test_bench_config_sampled_sequences():
    import bench
    L, E, H, S, B = bench.CONFIGS["small"]
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16")
    layers = [nnt_inputs.make_params(E, seed=1234, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    st = model.BlockStack(sc, layers)
    st.enable_graph()
    x = nnt_inputs.make_x(E, S, 0, B, seed=1000)
    r = nnt_inputs.make_r(E, S, 0, B, seed=1000)
    st.train_step(dev(x), dev(r))
    torch.cuda.synchronize()
    y = st.xs[-1]
    dx = st.dy[L % 2]  # backward ping-pongs between the two dy buffers, one flip per layer
    used = [_used(p) for p in layers]
    for j in (0, B - 1):
        xj, rj = x[j:j + 1], r[j:j + 1]
        yr, caches = dense.stack_fwd(used, xj, H)
        dxr, _ = dense.stack_bwd(used, caches, dense.probe_loss_grad(rj, B * S))
        close(host(y[j]), yr[0], 2e-2, j)
        close(host(dx[j]), dxr[0], 2e-2, j)


@pytest.mark.timeout(900)
def test_bench_config_full_gpt2_sampled_sequences():
    """The bench's default workload (full GPT-2 small: B=8, S=1024, 12 layers, V=50257, GPT-2 init,
    one CUDA-graph step): the per-token cross-entropy of sequences 0 and 7 against the oracle run
    on those sequences alone (the forward is independent across sequences)."""
    import bench
    L, E, H, S, B = bench.CONFIGS["small"]
    V = bench.VOCAB
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16")
    layers = [nnt_inputs.make_params(E, seed=1234, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    shell = nnt_inputs.make_shell_params(V, S, E, seed=1234, init="gpt2")
    gm = model.GPT2Model(sc, V, layers, shell)
    gm.enable_graph()
    tok = nnt_inputs.make_ids(V, S, 0, B, seed=1000)
    T = torch.as_tensor(tok).cuda()
    gm.train_step(T[:, :S].contiguous(), T[:, 1:].contiguous())
    torch.cuda.synchronize()
    rows = host(gm.loss_rows).reshape(B, S)
    om = dict(wte=bf16_round(shell["wte"]), wpe=shell["wpe"].astype(np.float64),
              lnf_g=shell["lnf_g"].astype(np.float64), lnf_b=shell["lnf_b"].astype(np.float64),
              blocks=[_used(p) for p in layers])
    for j in (0, B - 1):
        _, cache = dense.gpt2_fwd(om, tok[j:j + 1, :S], tok[j:j + 1, 1:], H)
        want, _ = dense.cross_entropy(cache["logits"], tok[j, 1:])
        close(rows[j], want, 2e-2, j)


@pytest.mark.timeout(1500)
def test_xl_bench_shape_block_every_gradient():
    """One GPT-2 XL block at the exact per-layer shapes the default bench times (E=1600, H=25, B=8,
    S=1024: T = 8192 tokens, so the dW GEMMs run K = 8192, the N = 1600 GEMMs their narrow tail
    tiles after the full ones, the MN-major operands the blocked TMA maps), GPT-2 init, one
    CUDA-graph training step (forward, probe loss, backward, Adam): y, dx, every parameter
    gradient and the Adam step against the fp64 oracle on the same batch, norm-wise and
    element-wise (reading R32)."""
    import bench
    _, E, H, S, B = bench.CONFIGS["xl"]
    assert (E, H, S, B) == (1600, 25, 1024, 8)
    sc = model.StackConfig(L=1, E=E, H=H, S=S, B=B, dtype="bf16")
    layers = [nnt_inputs.make_params(E, seed=2468, layer=0, init="gpt2", n_layers=48)]
    st = model.BlockStack(sc, layers)
    st.enable_graph()
    x = nnt_inputs.make_x(E, S, 0, B, seed=1357)
    r = nnt_inputs.make_r(E, S, 0, B, seed=1357)
    w0 = {n: host(v).astype(np.float64) for n, v in st.params_of(0).items()}
    st.train_step(dev(x), dev(r))
    torch.cuda.synchronize()
    got_y, got_dx = host(st.xs[-1]), host(st.dy[1])  # L = 1: backward's dx lands in dy[1]
    got_g = {n: host(v) for n, v in st.grads_of(0).items()}
    got_w = {n: host(v).astype(np.float64) for n, v in st.params_of(0).items()}
    used = _used(layers[0])
    del st, layers
    torch.cuda.empty_cache()
    y_ref, cache = dense.block_fwd(used, x, H)
    close(got_y, y_ref, 2e-2, "y")
    dx_ref, g_ref = dense.block_bwd(used, cache, dense.probe_loss_grad(r, B * S))
    del cache
    close(got_dx, dx_ref, 2e-2, "dx")
    for n, gv in got_g.items():
        if n == "b_qkv":  # the key-bias gradient is exactly zero in exact arithmetic (reading R22)
            close(np.delete(gv, np.s_[E:2 * E]), np.delete(g_ref[n], np.s_[E:2 * E]), 2e-2, n)
            assert np.abs(gv[E:2 * E]).max() <= 1e-3 * np.abs(g_ref[n]).max()
        else:
            close(gv, g_ref[n], 2e-2, n)
    # Adam step 1 from zero moments: w1 - w0 = -lr * g / (|g| + eps) elementwise (sign step), so
    # compare the update on the elements whose oracle gradient is clearly non-zero
    for n in got_w:
        w1, _, _ = dense.adam_step(w0[n], g_ref[n], np.zeros_like(w0[n]), np.zeros_like(w0[n]), 1)
        keep = np.abs(g_ref[n]) > 5e-2 * np.abs(g_ref[n]).max()
        if n == "b_qkv":
            keep[E:2 * E] = False
        d_got, d_want = (got_w[n] - w0[n])[keep], (w1 - w0[n])[keep]
        close(d_got, d_want, 2e-2, f"adam {n}")
