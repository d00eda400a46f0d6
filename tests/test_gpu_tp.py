"""Tensor-parallel block shards through the C ABI (nnt_block_tp_fwd / nnt_block_tp_bwd; SURVEY
§8(f) f2, reading R31) against the fp64 oracle.

R shards of one block run on the one GPU; the test itself plays the group's SUM reduction
between the stages (a torch sum of the shards' partial outputs), which is the exchange
tp.TPBlockStack does with NCCL.  y and dx must match the unsharded oracle block, and every
shard's gradients its slice of the oracle's gradients (tp.tp_shard).  fp32 path rel 1e-4,
bf16 path rel 2e-2 (north_star's tolerances).  The NCCL driver itself (TPBlockStack, world
size 1) is checked against the oracle over two training steps."""
import socket

import numpy as np
import pytest
import torch

import nnt_inputs
from oracle import dense
from gpu_util import close, close_update, bf16_round, dev, host, rel

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import model, nnt, tp


def _used(p, bf):
    return {k: (bf16_round(v) if (bf and k.startswith("w_")) else v.astype(np.float64)) for k, v in p.items()}


class _Shard:
    def __init__(self, cfg, sp, heads, ffn, add_bias, bf):
        self.tp = nnt.nnt_block_tp(heads, ffn, add_bias)
        self.t = {n: dev(v) for n, v in sp.items()}
        self.w16 = {n: dev(v, torch.bfloat16) for n, v in sp.items() if n.startswith("w_")} if bf else {}
        self.g = {n: torch.zeros_like(v) for n, v in self.t.items()}
        self.p = nnt.nnt_block_params()
        for n in sp:
            src = self.w16[n] if n in self.w16 else self.t[n]
            setattr(self.p, n, src.data_ptr())
        self.gr = nnt.nnt_block_grads()
        for n in sp:
            setattr(self.gr, n, self.g[n].data_ptr())
        sb, kb = nnt.nnt_block_tp_workspace_size(cfg, self.tp)
        self.saved = torch.empty(sb, device="cuda", dtype=torch.uint8)
        self.scratch = torch.zeros(kb, device="cuda", dtype=torch.uint8)


def _run_shards(E, H, S, B, R, dtype, tile, seed=11, fused=False):
    """fused: the partial-producing GEMMs scatter their rows into the owners' receive slots and the
    SUM is completed by nnt_tp_signal / nnt_tp_reduce_gather / nnt_tp_wait (R35), with the R ranks
    standing in this process (their buffers plain allocations); else the test sums the partials.
    Both sum in rank order (p0 + p1 + ...), so the two runs must agree bitwise."""
    bf = dtype == "bf16"
    sc = model.StackConfig(L=1, E=E, H=H, S=S, B=B, tile_e=tile, tile_f=tile, tile_s=tile, tile_t=tile,
                           dtype=dtype)
    cfg = sc.block_cfg()
    p = nnt_inputs.make_params(E, seed=seed, init="parity")
    shards = [_Shard(cfg, tp.tp_shard(p, H, R, r), H // R, 4 * E // R, 1 if r == 0 else 0, bf) for r in range(R)]
    x = nnt_inputs.make_x(E, S, 0, B, seed=seed + 1)
    dy = nnt_inputs.make_r(E, S, 0, B, seed=seed + 1) / (B * S)
    X, DY = dev(x), dev(dy)
    x1 = [torch.full_like(X, float("nan")) for _ in range(R)]
    y = [torch.full_like(X, float("nan")) for _ in range(R)]
    dh = [torch.full_like(X, float("nan")) for _ in range(R)]
    dx = [torch.empty_like(X) for _ in range(R)]
    T = B * S
    if fused:
        rows_per = -(-T // R)
        recv = [torch.full((R, rows_per, E), float("nan"), device="cuda") for _ in range(R)]
        flags = [torch.zeros(2 * nnt.NNT_TP_MAX, device="cuda", dtype=torch.int32) for _ in range(R)]
        comms = [nnt.make_tp_comm(R, r, T, E, recv, flags) for r in range(R)]
        for r, sh in enumerate(shards):
            sh.tp.comm = nnt.C.pointer(comms[r])
        epoch = [0]

    def allsum(bufs):
        if fused:  # every rank's GEMMs have scattered; the ranks complete the SUM in phases
            epoch[0] += 1
            for r in range(R):
                nnt.nnt_tp_signal(comms[r], epoch[0], 0)
            for r in range(R):
                nnt.nnt_tp_reduce_gather(comms[r], bufs, epoch[0])
            for r in range(R):
                nnt.nnt_tp_signal(comms[r], epoch[0], 1)
            for r in range(R):
                nnt.nnt_tp_wait(comms[r], epoch[0])
            return
        s = bufs[0].clone()
        for b in bufs[1:]:
            s += b
        for b in bufs:
            b.copy_(s)

    for st in (0, 1):
        for r, sh in enumerate(shards):
            nnt.nnt_block_tp_fwd(cfg, sh.tp, sh.p, st, X, x1[r], y[r] if st else None, sh.saved, sh.scratch)
        allsum(x1 if st == 0 else y)
    for st in (0, 1, 2):
        for r, sh in enumerate(shards):
            nnt.nnt_block_tp_bwd(cfg, sh.tp, sh.p, st, X, x1[r], sh.saved, sh.scratch, DY, dh[r],
                                 dx[r] if st == 2 else None, sh.gr, 0)
        if st < 2:
            allsum(dh)
    torch.cuda.synchronize()
    used = _used(p, bf)
    y_ref, cache = dense.block_fwd(used, x, H)
    dx_ref, g_ref = dense.block_bwd(used, cache, dy)
    return shards, y, dx, y_ref, dx_ref, g_ref


@pytest.mark.parametrize("E,H,S,B,R,dtype,tile,tol", [
    (64, 4, 32, 2, 1, "f32", 16, 1e-4),
    (64, 4, 32, 2, 2, "f32", 16, 1e-4),
    (64, 4, 32, 2, 4, "f32", 16, 1e-4),
    (256, 4, 256, 2, 2, "bf16", 1024, 2e-2),
    (256, 4, 256, 2, 4, "bf16", 1024, 2e-2),
    (768, 12, 128, 2, 3, "bf16", 1024, 2e-2),
], ids=["f32-R1", "f32-R2", "f32-R4", "bf16-R2", "bf16-R4", "bf16-E768-R3"])
def test_tp_shards_match_oracle(E, H, S, B, R, dtype, tile, tol):
    shards, y, dx, y_ref, dx_ref, g_ref = _run_shards(E, H, S, B, R, dtype, tile)
    for r in range(R):
        close(host(y[r]), y_ref, tol, r)
        close(host(dx[r]), dx_ref, tol, r)
        want = tp.tp_shard(g_ref, H, R, r)
        for n, gv in shards[r].g.items():
            close(host(gv), want[n], tol, (r, n))
    if R > 1:  # replicated parameters' gradients are bitwise equal on every shard
        for n in ("ln1_g", "ln1_b", "b_o", "ln2_g", "ln2_b", "b_pr"):
            for r in range(1, R):
                assert torch.equal(shards[r].g[n], shards[0].g[n]), (n, r)


@pytest.mark.parametrize("E,H,S,B,R,dtype,tile", [
    (64, 4, 32, 2, 1, "f32", 16), (64, 4, 32, 2, 4, "f32", 16), (96, 6, 32, 2, 3, "f32", 16),
    (256, 4, 256, 2, 2, "bf16", 1024), (768, 12, 128, 2, 3, "bf16", 1024),
], ids=["f32-R1", "f32-R4", "f32-R3-ragged", "bf16-R2", "bf16-E768-R3-ragged"])
def test_tp_fused_reduction_equals_summed_partials(E, H, S, B, R, dtype, tile):
    """R35: the partial-producing GEMMs (out-projection, projection, FC-dX, QKV-dX) write their
    rows straight into the owners' receive slots and the owners sum them in rank order and
    gather the sums to every rank: y, dx and every gradient bitwise equal to the run whose
    partials the test sums in the same order (T = 64 / 256 rows over 3 ranks: a short last
    owner), and within tolerance of the oracle."""
    a = _run_shards(E, H, S, B, R, dtype, tile, fused=True)
    b = _run_shards(E, H, S, B, R, dtype, tile, fused=False)
    for r in range(R):
        assert torch.equal(a[1][r], b[1][r]) and torch.equal(a[2][r], b[2][r]), r
        for n in a[0][r].g:
            assert torch.equal(a[0][r].g[n], b[0][r].g[n]), (r, n)
    tol = 1e-4 if dtype == "f32" else 2e-2
    close(host(a[1][0]), a[3], tol, "y")
    close(host(a[2][0]), a[4], tol, "dx")


def test_tp_argument_errors():
    sc = model.StackConfig(L=1, E=64, H=4, S=32, B=2, tile_e=16, tile_f=16, tile_s=16, tile_t=16, dtype="f32")
    cfg = sc.block_cfg()
    with pytest.raises(nnt.NNTError):
        nnt.nnt_block_tp_workspace_size(cfg, nnt.nnt_block_tp(5, 64, 1))  # more heads than H
    with pytest.raises(nnt.NNTError):
        nnt.nnt_block_tp_workspace_size(cfg, nnt.nnt_block_tp(2, 60, 1))  # ffn not a multiple of 8
    with pytest.raises(nnt.NNTError):
        nnt.nnt_block_tp_workspace_size(cfg, nnt.nnt_block_tp(2, 64, 2))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_tp_stack_fused_world1_equals_nccl():
    """TPBlockStack with the fused peer-memory SUMs (R35) on a group of one rank: two training
    steps bitwise equal to the NCCL-reduced stack (bf16, 2 layers)."""
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        E, H, S, B, L = 256, 4, 256, 2, 2
        sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16", lr=1e-3)
        layers = [nnt_inputs.make_params(E, seed=23, layer=l, n_layers=L) for l in range(L)]
        runs = []
        for fused in (True, False):
            st = tp.TPBlockStack(sc, layers, dist.group.WORLD, fused=fused)
            for t in (1, 2):
                x = dev(nnt_inputs.make_x(E, S, 0, B, seed=40 + t))
                r = dev(nnt_inputs.make_r(E, S, 0, B, seed=40 + t))
                st.train_step(x, r)
            torch.cuda.synchronize()
            runs.append((st.w.clone(), st.g.clone(), st.xs[-1].clone(), st.loss.clone()))
        for a, b in zip(*runs):
            assert torch.equal(a, b)
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_tp_stack_nccl_world1_two_adam_steps():
    """TPBlockStack (NCCL group of one rank, 2 layers, fp32): two training steps (forward,
    probe loss, backward with the four reductions per block, Adam) vs the oracle."""
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        E, H, S, B, L = 64, 4, 32, 2, 2
        sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, tile_e=16, tile_f=16, tile_s=16, tile_t=16, dtype="f32",
                               lr=1e-2)
        layers = [nnt_inputs.make_params(E, seed=21, layer=l, n_layers=L) for l in range(L)]
        st = tp.TPBlockStack(sc, layers, dist.group.WORLD)
        P = [{k: v.astype(np.float64) for k, v in d.items()} for d in layers]
        mv = [{k: (np.zeros_like(v), np.zeros_like(v)) for k, v in d.items()} for d in P]
        for t in (1, 2):
            x = nnt_inputs.make_x(E, S, 0, B, seed=30 + t)
            r = nnt_inputs.make_r(E, S, 0, B, seed=30 + t)
            loss = st.train_step(dev(x), dev(r)).item()
            y, caches = dense.stack_fwd(P, x, H)
            want = dense.probe_loss(y, r, B * S)
            _, g = dense.stack_bwd(P, caches, dense.probe_loss_grad(r, B * S))
            assert abs(loss - want) <= 1e-4 * abs(want), t
            torch.cuda.synchronize()
            for l in range(L):  # this step's gradients (taken at the GPU's parameters) vs the oracle's
                for n, gv in st.grads_of(l).items():
                    if n != "b_qkv":
                        close(host(gv), g[l][n], 1e-4, (t, l, n))
            for l in range(L):
                for n in P[l]:
                    P[l][n], m1, v1 = dense.adam_step(P[l][n], g[l][n], *mv[l][n], t, lr=1e-2)
                    mv[l][n] = (m1, v1)
        torch.cuda.synchronize()
        # b_k's gradient is zero in exact arithmetic (softmax is shift invariant), so its Adam
        # steps are +-lr driven by rounding noise on either side: only bounded, not compared
        for l in range(L):
            for n, wv in st.params_of(l).items():
                got, want, w0 = host(wv).ravel(), P[l][n].ravel(), layers[l][n].ravel().astype(np.float64)
                rms = np.sqrt(mv[l][n][1]).ravel()
                if n == "b_qkv":
                    assert np.abs(got[E:2 * E] - want[E:2 * E]).max() <= 4 * 1e-2 * 1.01, l
                    keep = np.r_[0:E, 2 * E:3 * E]
                    got, want, w0, rms = got[keep], want[keep], w0[keep], rms[keep]
                close_update(got - w0, want - w0, want, rms, 1e-4, (l, n), elementwise=False)
    finally:
        if own:
            dist.destroy_process_group()
