"""Data-parallel semantics on the oracle (CPU): batch tiles partitioned across
ranks + SUM of per-rank gradients equals the full-batch gradient (reading R14,
PAPER.md:124-127 "gradients of the same matrix of parameters from different
devices are accumulated").  Covered two ways: an in-process ordered sum and a
real world_size-2 gloo all_reduce."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nnt_inputs
from oracle import dense, tiled

E, H, S, NB = 16, 2, 8, 4


def _grads_for(rank, R, seed_p=3, seed_x=4):
    b0, b1 = tiled.partition(NB, R, rank)
    params = nnt_inputs.make_params(E, seed=seed_p)
    x = nnt_inputs.make_x(E, S, b0, b1, seed=seed_x)
    r = nnt_inputs.make_r(E, S, b0, b1, seed=seed_x)
    y, cache = dense.block_fwd(params, x, H)
    _, grads = dense.block_bwd(params, cache, dense.probe_loss_grad(r, NB * S))
    return grads


def test_partitioned_sum_equals_full_batch():
    full = _grads_for(0, 1)
    for R in (2, 3, 4):
        parts = [_grads_for(r, R) for r in range(R)]
        for k in full:
            tot = sum(p[k] for p in parts)
            assert np.linalg.norm(tot - full[k]) <= 1e-12 * np.linalg.norm(full[k]), (R, k)


def test_inputs_identical_per_sequence_across_partitions():
    whole = nnt_inputs.make_x(E, S, 0, NB)
    for R in (2, 4):
        for r in range(R):
            b0, b1 = tiled.partition(NB, R, r)
            assert np.array_equal(nnt_inputs.make_x(E, S, b0, b1), whole[b0:b1])


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
    g = _grads_for(rank, world)
    flat = torch.tensor(np.concatenate([g[k].ravel() for k in dense.PARAM_NAMES]))
    dist.all_reduce(flat)
    if rank == 0:
        out.put(flat.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_allreduce_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _grads_for(0, 1)
    ref = np.concatenate([full[k].ravel() for k in dense.PARAM_NAMES])
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
