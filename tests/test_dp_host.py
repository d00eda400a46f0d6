"""Host logic of the DP path (CPU, gloo, world size 2): the flat parameter / gradient
layout and its all-reduce buckets (model.flat_layout), the batch-tile partition
(nnt_partition through the C ABI), and a bucket-by-bucket SUM all-reduce in
backward-completion order, as BlockStack.backward issues it on the GPU
(readings R14, R17: integer bookkeeping bit-exact across ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nnt_inputs
from oracle import dense

E, H, S, NB, L = 16, 2, 8, 4, 2


def _layout():
    from paper_2504_13236_b200 import model
    return model.flat_layout(L, E)


def test_flat_layout_buckets_cover_and_align():
    from paper_2504_13236_b200 import model
    for (LL, EE) in ((1, 64), (12, 768), (36, 1280), (48, 1600), (1, 8192)):
        offsets, buckets, numel = model.flat_layout(LL, EE)
        shapes = model.param_shapes(EE)
        # buckets tile [0, numel) contiguously, in backward-completion order
        assert buckets[0][2] == 0 and buckets[-1][3] == numel
        for a, b in zip(buckets, buckets[1:]):
            assert a[3] == b[2]
        assert [(l, si) for l, si, _, _ in buckets] == [(l, si) for l in range(LL - 1, -1, -1) for si in range(4)]
        for l in range(LL):
            for si, names in enumerate(model.SETS):
                b0, b1 = [(x[2], x[3]) for x in buckets if x[0] == l and x[1] == si][0]
                for n in names:
                    o, k = offsets[l][n]
                    assert o % model.ALIGN == 0 and b0 <= o and o + k <= b1
                    assert k == int(np.prod(shapes[n]))
        # no two tensors overlap
        spans = sorted(v for d in offsets for v in d.values())
        for (o0, k0), (o1, _) in zip(spans, spans[1:]):
            assert o0 + k0 <= o1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(b0, b1, layers):
    x = nnt_inputs.make_x(E, S, b0, b1, seed=11)
    r = nnt_inputs.make_r(E, S, b0, b1, seed=11)
    y, caches = dense.stack_fwd(layers, x, H)
    _, grads = dense.stack_bwd(layers, caches, dense.probe_loss_grad(r, NB * S))
    return grads


def _flat(grads, offsets, numel):
    buf = np.zeros(numel)
    for l, d in enumerate(offsets):
        for n, (o, k) in d.items():
            buf[o:o + k] = grads[l][n].ravel()
    return buf


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_13236_b200 import nnt
    offsets, buckets, numel = _layout()
    # the layout is identical on every rank (bit-exact)
    mine = torch.tensor([v for l, si, b0, b1 in buckets for v in (l, si, b0, b1)], dtype=torch.int64)
    allb = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allb, mine)
    same = all(torch.equal(allb[0], t) for t in allb)
    b0, b1 = nnt.nnt_partition(NB, world, rank)
    layers = [nnt_inputs.make_params(E, seed=5, layer=l, n_layers=L) for l in range(L)]
    g = torch.tensor(_flat(_grads(b0, b1, layers), offsets, numel))
    for (_, _, c0, c1) in buckets:  # backward-completion order, one collective per bucket
        v = g[c0:c1].clone()
        dist.all_reduce(v)
        g[c0:c1] = v
    if rank == 0:
        out.put((same, (b0, b1), g.numpy()))
    else:
        out.put((same, (b0, b1), None))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_bucketed_allreduce_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[0] for r in res)
    parts = sorted(r[1] for r in res)
    assert parts == [(0, NB // 2), (NB // 2, NB)]  # floor(r n / R) partition, covering the batch
    got = [r[2] for r in res if r[2] is not None][0]
    offsets, buckets, numel = _layout()
    layers = [nnt_inputs.make_params(E, seed=5, layer=l, n_layers=L) for l in range(L)]
    ref = _flat(_grads(0, NB, layers), offsets, numel)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
