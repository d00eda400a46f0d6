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


def test_zero_shards_partition():
    """ZeRO-1 ownership: per bucket, the world's owned slices tile the (padded) bucket exactly,
    ALIGN-aligned, and the compact state offsets pack each rank's slices back to back."""
    from paper_2504_13236_b200 import model
    for (LL, EE, R) in ((2, 16, 2), (12, 768, 8), (48, 1600, 4), (1, 8192, 3)):
        offsets, buckets, numel = model.flat_layout(LL, EE, shards=R)
        _, _, numel1 = model.flat_layout(LL, EE)
        assert numel >= numel1 and numel % (R * model.ALIGN) == 0
        for l in range(LL):  # the tensors still sit inside their buckets
            for si, names in enumerate(model.SETS):
                b0, b1 = [(x[2], x[3]) for x in buckets if x[0] == l and x[1] == si][0]
                for n in names:
                    o, k = offsets[l][n]
                    assert b0 <= o and o + k <= b1
        owned = [model.zero_shards(buckets, R, r) for r in range(R)]
        for r, (sh, nst) in enumerate(owned):
            assert nst * R == numel
            c = 0
            for (_, _, b0, b1) in buckets:
                s0, s1, cc = sh[b0]
                assert cc == c and s0 % model.ALIGN == 0 and s1 - s0 == (b1 - b0) // R
                assert s0 == b0 + r * (s1 - s0)
                c += s1 - s0
        for (_, _, b0, b1) in buckets:
            cover = sorted((owned[r][0][b0][0], owned[r][0][b0][1]) for r in range(R))
            assert cover[0][0] == b0 and cover[-1][1] == b1
            assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
        # the gather regions (bf16 shadows of the GEMM weight, fp32 small parameters): each a
        # multiple of R * ALIGN, the weight alone in the first, the rest in the second
        for b in buckets:
            l, si, b0, b1 = b
            (r0, mid, w0), (m1, r1, w1) = model.bucket_regions(offsets, b, R)
            assert (r0, r1, m1, w0, w1) == (b0, b1, mid, True, False)
            assert (mid - b0) % (R * model.ALIGN) == 0 and (b1 - mid) % (R * model.ALIGN) == 0
            o, k = offsets[l][model.SETS[si][0]]
            assert o == b0 and o + k <= mid
            assert all(mid <= offsets[l][n][0] for n in model.SETS[si][1:])
        regions = [r[:2] for b in buckets for r in model.bucket_regions(offsets, b, R)]
        for r in range(R):
            sh, nst = model.zero_shards(regions, R, r)
            assert nst * R == numel and all(s1 - s0 == (e - a) // R for (a, e), (s0, s1, _) in
                                             zip(regions, [sh[a] for a, _ in regions]))
    offsets1, buckets1, _ = model.flat_layout(2, 16)
    assert model.bucket_regions(offsets1, buckets1[0], 1) == [(buckets1[0][2], buckets1[0][3], True)]


def _zero_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_13236_b200 import model, nnt
    offsets, buckets, numel = model.flat_layout(L, E, shards=world)
    sh, nst = model.zero_shards(buckets, world, rank)
    b0, b1 = nnt.nnt_partition(NB, world, rank)
    layers = [nnt_inputs.make_params(E, seed=5, layer=l, n_layers=L) for l in range(L)]
    w = torch.tensor(_flat(layers, offsets, numel))
    m, v = torch.zeros(nst, dtype=torch.float64), torch.zeros(nst, dtype=torch.float64)
    for t in (1, 2):  # two optimizer steps, the second on the first's updated replica
        P = [{n: w[o:o + k].numpy().reshape(layers[0][n].shape).copy() for n, (o, k) in offsets[l].items()}
             for l in range(L)]
        g = torch.tensor(_flat(_grads(b0, b1, P), offsets, numel))

        def update(s0, s1, c, t=t, g=g):
            n = s1 - s0
            w1, m1, v1 = dense.adam_step(w[s0:s1].numpy(), g[s0:s1].numpy(), m[c:c + n].numpy(),
                                         v[c:c + n].numpy(), t, weight_decay=0.01)
            w[s0:s1], m[c:c + n], v[c:c + n] = torch.tensor(w1), torch.tensor(m1), torch.tensor(v1)

        for (_, _, c0, c1) in buckets:
            s0, s1, c = sh[c0]
            model.zero1_bucket(g, w, c0, c1, s0, s1, None, lambda a, b, c=c: update(a, b, c))
    out.put((rank, w.numpy() if rank == 0 else None, nst))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_zero1_equals_replicated_adam():
    """The ZeRO-1 bucket step (model.zero1_bucket, the same host code BlockStack runs on NCCL):
    reduce-scatter by owned slice, AdamW on the owned slice with half-size state, all-gather of
    the updated parameters -- two steps on two ranks equal two replicated full-batch AdamW
    steps of the oracle (fp64)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zero_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2504_13236_b200 import model
    offsets, buckets, numel = model.flat_layout(L, E, shards=2)
    assert all(r[2] * 2 == numel for r in res)
    got = [r[1] for r in res if r[1] is not None][0]
    layers = [nnt_inputs.make_params(E, seed=5, layer=l, n_layers=L) for l in range(L)]
    P = [{n: layers[l][n].astype(np.float64) for n in layers[l]} for l in range(L)]
    st = [{n: (np.zeros_like(p), np.zeros_like(p)) for n, p in d.items()} for d in P]
    for t in (1, 2):
        g = _grads(0, NB, P)
        for l in range(L):
            for n in P[l]:
                P[l][n], m1, v1 = dense.adam_step(P[l][n], g[l][n], *st[l][n], t, weight_decay=0.01)
                st[l][n] = (m1, v1)
    ref = _flat(P, offsets, numel)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
