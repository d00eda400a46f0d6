"""Full-gradient, element-wise parity against the fp64 oracle (VERDICT r1 "next" #1).

* The exact step bench.py times by default for GPT-2 small (12 layers, E=768, H=12, B=8, S=1024,
  V=50257, GPT-2 init, one CUDA-graph training step): EVERY gradient tensor (all 12 layers' W, b,
  gamma, beta, plus wte, wpe, lnf) against the oracle's full-batch gradient, norm-wise and
  element-wise (gpu_util.close), and the Adam update of every parameter against the oracle's Adam
  applied to the same gradient.  The oracle runs one sequence at a time and sums the gradients
  (every parameter gradient is a sum over tokens; t_global = B*S scales each sequence's share).
* Multi-step training of the full model: at every step the gradients must equal the oracle's
  gradients AT THE PARAMETERS THE GPU HELD BEFORE THAT STEP (so a gradient buffer that is not
  reset between steps -- the r1 wpe bug -- fails at step 2), eager and graph-captured; on the fp32
  path the whole 3-step parameter trajectory is compared with the oracle's too.
"""
import numpy as np
import pytest
import torch

import nnt_inputs
from oracle import dense
from gpu_util import bf16_round, close, close_update, host

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import model

SHELL = ("wte", "wpe", "lnf_g", "lnf_b")


def _oracle_model(gm, bf16):
    """The parameters the GPU computes with, read back from the device: bf16-rounded weight matrices
    and token table on the bf16 path (the GEMM operands are the bf16 shadows), fp32 otherwise."""
    rnd = bf16_round if bf16 else (lambda a: np.asarray(a, np.float64))
    sh = {k: host(v) for k, v in gm.params().items()}
    om = dict(wte=rnd(sh["wte"]), wpe=sh["wpe"], lnf_g=sh["lnf_g"], lnf_b=sh["lnf_b"], blocks=[])
    for l in range(gm.cfg.L):
        p = {k: host(v) for k, v in gm.stack.params_of(l).items()}
        om["blocks"].append({k: (rnd(v) if k.startswith("w_") else v) for k, v in p.items()})
    return om, sh


def _oracle_grads(om, tok, S, H, per_sequence=False):
    """dense.gpt2_bwd of the mean CE over the whole batch; per_sequence=True sums sequence by
    sequence (identical math: the loss is a sum over tokens scaled by 1/T_global)."""
    B = tok.shape[0]
    if not per_sequence:
        loss, cache = dense.gpt2_fwd(om, tok[:, :S], tok[:, 1:], H)
        return loss, dense.gpt2_bwd(om, cache)
    total, acc = 0.0, None
    for j in range(B):
        lj, cache = dense.gpt2_fwd(om, tok[j:j + 1, :S], tok[j:j + 1, 1:], H)
        gj = dense.gpt2_bwd(om, cache, t_global=B * S)
        del cache
        total += lj * S / (B * S)
        if acc is None:
            acc = gj
        else:
            for k in SHELL:
                acc[k] += gj[k]
            for l, gl in enumerate(gj["blocks"]):
                for k in gl:
                    acc["blocks"][l][k] += gl[k]
    return total, acc


def _compare_grads(gm, g, tol, tag):
    got = {k: host(v) for k, v in gm.grads().items()}
    for k in SHELL:
        close(got[k], g[k], tol, f"{tag} {k}")
    for l in range(gm.cfg.L):
        for k, v in gm.stack.grads_of(l).items():
            if k == "b_qkv":  # the key-bias third is exactly zero in exact arithmetic (R22)
                E = gm.cfg.E
                gv, wv = host(v), g["blocks"][l][k]
                close(np.concatenate([gv[:E], gv[2 * E:]]), np.concatenate([wv[:E], wv[2 * E:]]), tol,
                      f"{tag} L{l} b_qkv(q,v)")
                assert np.abs(gv[E:2 * E]).max() <= tol * np.abs(wv).max() + 1e-30, f"{tag} L{l} key bias"
                continue
            close(host(v), g["blocks"][l][k], tol, f"{tag} L{l} {k}")


def _adam_delta_check(gm, w0_shell, w0_blocks, t, tol=1e-4):
    """Adam on the GPU vs dense.adam_step applied to the GPU's own gradient (first step: m = v = 0).
    Decoupled from gradient noise: at step 1 Adam's update is ~lr*sign(g), so comparing it with the
    oracle-gradient update would test the sign of near-zero gradient entries, not the kernel."""
    c = gm.cfg
    assert t == 1
    kw = dict(lr=c.lr, beta1=c.beta1, beta2=c.beta2, eps=c.eps)
    for k, v in gm.params().items():
        g = host(gm.grads()[k])
        w1, _, _ = dense.adam_step(w0_shell[k], g, np.zeros_like(g), np.zeros_like(g), t, **kw)
        close(host(v) - w0_shell[k], w1 - w0_shell[k], tol, f"adam {k}")
    for l in range(c.L):
        gr = gm.stack.grads_of(l)
        for k, v in gm.stack.params_of(l).items():
            g = host(gr[k])
            w1, _, _ = dense.adam_step(w0_blocks[l][k], g, np.zeros_like(g), np.zeros_like(g), t, **kw)
            close(host(v) - w0_blocks[l][k], w1 - w0_blocks[l][k], tol, f"adam L{l} {k}")


@pytest.mark.timeout(1800)
def test_bench_step_every_gradient_and_adam():
    import bench
    L, E, H, S, B = bench.CONFIGS["small"]
    V = bench.VOCAB
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16")
    layers = [nnt_inputs.make_params(E, seed=1234, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    shell = nnt_inputs.make_shell_params(V, S, E, seed=1234, init="gpt2")
    gm = model.GPT2Model(sc, V, layers, shell)
    del layers, shell
    gm.enable_graph()
    om, w0_shell = _oracle_model(gm, bf16=True)
    w0_blocks = [{k: host(v) for k, v in gm.stack.params_of(l).items()} for l in range(L)]
    tok = nnt_inputs.make_ids(V, S, 0, B, seed=1000)
    T = torch.as_tensor(tok).cuda()
    loss = gm.train_step(T[:, :S].contiguous(), T[:, 1:].contiguous()).item()
    torch.cuda.synchronize()
    _adam_delta_check(gm, w0_shell, w0_blocks, 1)
    want, g = _oracle_grads(om, tok, S, H, per_sequence=True)
    assert abs(loss - want) <= 2e-2 * abs(want)
    _compare_grads(gm, g, 2e-2, "bench-step")


@pytest.mark.timeout(900)
@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
@pytest.mark.parametrize("cfg", ["f32-tiny", "bf16-small-vocab"])
def test_gpt2_multistep_gradients_vs_oracle(cfg, graph):
    if cfg == "f32-tiny":
        V, E, H, S, B, L, dtype, tol, tile = 128, 64, 2, 32, 2, 2, "f32", 1e-4, 16
    else:
        V, E, H, S, B, L, dtype, tol, tile = 50257, 768, 12, 128, 2, 2, "bf16", 2e-2, 1024
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype=dtype, tile_e=tile, tile_f=tile, tile_s=tile,
                           tile_t=tile)
    layers = [nnt_inputs.make_params(E, seed=9, layer=l, init="parity", n_layers=L) for l in range(L)]
    shell = nnt_inputs.make_shell_params(V, S, E, seed=10, init="parity")
    gm = model.GPT2Model(sc, V, layers, shell)
    if graph:
        gm.enable_graph()
    bf16 = dtype == "bf16"
    # fp32: the oracle's own 3-step Adam trajectory from the same initial parameters
    traj = {k: v.astype(np.float64) for k, v in shell.items()}
    traj["blocks"] = [{k: v.astype(np.float64) for k, v in p.items()} for p in layers]
    mom = {"shell": {k: (np.zeros_like(v), np.zeros_like(v)) for k, v in traj.items() if k != "blocks"},
           "blocks": [{k: (np.zeros_like(v), np.zeros_like(v)) for k, v in p.items()} for p in traj["blocks"]]}
    for t in range(1, 4):
        om, _ = _oracle_model(gm, bf16)
        tok = nnt_inputs.make_ids(V, S, 0, B, seed=300 + t)
        Tt = torch.as_tensor(tok).cuda()
        loss = gm.train_step(Tt[:, :S].contiguous(), Tt[:, 1:].contiguous()).item()
        torch.cuda.synchronize()
        want, g = _oracle_grads(om, tok, S, H)
        assert abs(loss - want) <= tol * abs(want), (t, loss, want)
        _compare_grads(gm, g, tol, f"step{t}")
        if not bf16:
            _, gt = _oracle_grads(traj, tok, S, H)
            for k in SHELL:
                m, v = mom["shell"][k]
                traj[k], m, v = dense.adam_step(traj[k], gt[k], m, v, t)
                mom["shell"][k] = (m, v)
            for l in range(L):
                for k in traj["blocks"][l]:
                    m, v = mom["blocks"][l][k]
                    traj["blocks"][l][k], m, v = dense.adam_step(traj["blocks"][l][k], gt["blocks"][l][k], m, v, t)
                    mom["blocks"][l][k] = (m, v)
    if not bf16:  # the trajectory: parameter change over 3 steps vs the oracle's, key bias excluded (R22)
        for k, v in gm.params().items():
            close_update(host(v) - shell[k], traj[k] - shell[k], traj[k], np.sqrt(mom["shell"][k][1]), 1e-4,
                         f"traj {k}", elementwise=False)
        for l in range(L):
            for k, v in gm.stack.params_of(l).items():
                got, want = host(v) - layers[l][k], traj["blocks"][l][k] - layers[l][k]
                w1, rms = traj["blocks"][l][k], np.sqrt(mom["blocks"][l][k][1])
                if k == "b_qkv":
                    got, want, w1, rms = (np.delete(a, np.s_[E:2 * E]) for a in (got, want, w1, rms))
                close_update(got, want, w1, rms, 1e-4, f"traj L{l} {k}", elementwise=False)
