"""Host logic of the tensor-parallel block (reading R31): the shard slicing
(tp.tp_shard / tp_unshard) and the stage / reduction schedule of nnt_block_tp_fwd / _bwd,
executed with the fp64 oracle's primitives on R gloo ranks (CPU) and checked against the
unsharded oracle block.  The schedule written out here is the one nnt.h documents and
tp.TPBlockStack issues: x1 and y reduced in the forward, dL/dh2 and dL/dh1 in the backward;
b_o, b_pr and the residuals added on rank 0 only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nnt_inputs
from oracle import dense

E, H, S, B = 32, 4, 8, 2


def test_shard_unshard_roundtrip_and_shapes():
    from paper_2504_13236_b200 import tp
    p = nnt_inputs.make_params(E, seed=3)
    for R in (1, 2, 4):
        sh = [tp.tp_shard(p, H, R, r) for r in range(R)]
        for s in sh:
            assert {n: v.shape for n, v in s.items()} == tp.shard_shapes(E, H, R)
        back = tp.tp_unshard(sh, H)
        for n in p:
            assert np.array_equal(back[n], p[n]), (R, n)
    # the q, k and v rows of one head go to the same rank
    s = tp.tp_shard(p, H, 2, 1)
    Dh = E // H
    assert np.array_equal(s["w_qkv"][:2 * Dh], p["w_qkv"][2 * Dh:4 * Dh])
    assert np.array_equal(s["w_qkv"][2 * Dh:4 * Dh], p["w_qkv"][E + 2 * Dh:E + 4 * Dh])
    assert np.array_equal(s["w_qkv"][4 * Dh:], p["w_qkv"][2 * E + 2 * Dh:2 * E + 4 * Dh])


def _staged_block(P, x, dy, hl, rank, allsum):
    """One shard's forward and backward in the stage order of nnt.h (oracle primitives)."""
    z = lambda n: np.zeros(P[n].shape[0])  # noqa: E731
    add = rank == 0
    # fwd stage 0
    h1, mu1, r1 = dense.layernorm_fwd(x, P["ln1_g"], P["ln1_b"])
    qkv = dense.linear_fwd(h1, P["w_qkv"], P["b_qkv"])
    o, p = dense.attention_core_fwd(qkv, hl)
    x1 = dense.linear_fwd(o, P["w_o"], P["b_o"] if add else z("b_o")) + (x if add else 0)
    x1 = allsum(x1)
    # fwd stage 1
    h2, mu2, r2 = dense.layernorm_fwd(x1, P["ln2_g"], P["ln2_b"])
    u = dense.linear_fwd(h2, P["w_fc"], P["b_fc"])
    g = dense.gelu(u)
    y = dense.linear_fwd(g, P["w_pr"], P["b_pr"] if add else z("b_pr")) + (x1 if add else 0)
    y = allsum(y)
    # bwd stage 0
    gr = {}
    dg, gr["w_pr"], gr["b_pr"] = dense.linear_bwd(dy, g, P["w_pr"])
    du = dense.gelu_bwd(u, dg)
    dh2, gr["w_fc"], gr["b_fc"] = dense.linear_bwd(du, h2, P["w_fc"])
    dh2 = allsum(dh2)
    # bwd stage 1
    dx1_ln, gr["ln2_g"], gr["ln2_b"] = dense.layernorm_bwd(dh2, x1, P["ln2_g"], mu2, r2)
    dx1 = dy + dx1_ln
    do, gr["w_o"], gr["b_o"] = dense.linear_bwd(dx1, o, P["w_o"])
    dqkv = dense.attention_core_bwd(do, qkv, p, hl)
    dh1, gr["w_qkv"], gr["b_qkv"] = dense.linear_bwd(dqkv, h1, P["w_qkv"])
    dh1 = allsum(dh1)
    # bwd stage 2
    dx_ln, gr["ln1_g"], gr["ln1_b"] = dense.layernorm_bwd(dh1, x, P["ln1_g"], mu1, r1)
    return y, dx1 + dx_ln, gr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_13236_b200 import tp

    def allsum(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    p = nnt_inputs.make_params(E, seed=3)
    P = {n: v.astype(np.float64) for n, v in tp.tp_shard(p, H, world, rank).items()}
    x = nnt_inputs.make_x(E, S, 0, B, seed=4).astype(np.float64)
    dy = nnt_inputs.make_r(E, S, 0, B, seed=4).astype(np.float64) / (B * S)
    y, dx, gr = _staged_block(P, x, dy, H // world, rank, allsum)
    out.put((rank, y, dx, gr))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_gloo_tp_schedule_equals_unsharded_block(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2504_13236_b200 import tp
    p = nnt_inputs.make_params(E, seed=3)
    x = nnt_inputs.make_x(E, S, 0, B, seed=4)
    dy = nnt_inputs.make_r(E, S, 0, B, seed=4).astype(np.float64) / (B * S)
    y_ref, cache = dense.block_fwd(p, x, H)
    dx_ref, g_ref = dense.block_bwd(p, cache, dy)
    for rank, y, dx, gr in res:
        # y and dx are replicated: every rank holds the full result
        assert np.allclose(y, y_ref, rtol=0, atol=1e-12 * np.abs(y_ref).max())
        assert np.allclose(dx, dx_ref, rtol=0, atol=1e-12 * np.abs(dx_ref).max())
        # each rank's gradients are exactly its slice of the full gradients
        want = tp.tp_shard(g_ref, H, world, rank)
        for n in want:
            assert np.allclose(gr[n], want[n], rtol=0, atol=1e-12 * max(np.abs(want[n]).max(), 1e-30)), (rank, n)
