"""The DP code path on one GPU: a world-size-1 NCCL process group makes BlockStack run the
data-parallel backward (bucket events from nnt_block_bwd, NCCL SUM all-reduce of each bucket
on the communication stream, Adam per bucket overlapping the rest of the backward pass),
eagerly and captured in a CUDA graph.  A one-rank SUM is the identity and Adam is elementwise,
so parameters, moments and losses must equal the single-GPU path bitwise (reading R17)."""
import os
import socket

import pytest
import torch

import nnt_inputs
from gpu_util import dev

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import model


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def _run(pg, graph, steps=3, zero=False):
    E, H, S, B, L = 768, 12, 256, 2, 2
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16", zero=zero)
    layers = [nnt_inputs.make_params(E, seed=9, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    st = model.BlockStack(sc, layers, process_group=pg)
    if graph:
        st.enable_graph()
    losses = []
    for t in range(steps):
        x = dev(nnt_inputs.make_x(E, S, 0, B, seed=70 + t))
        r = dev(nnt_inputs.make_r(E, S, 0, B, seed=70 + t))
        losses.append(st.train_step(x, r).item())
    torch.cuda.synchronize()
    return losses, st.w.clone(), st.m.clone(), st.v.clone(), st.w16.clone()


@pytest.mark.timeout(300)
def test_dp_path_world1_equals_single_gpu_bitwise(pg):
    ref = _run(None, graph=False)
    for graph in (False, True):
        got = _run(pg, graph=graph)
        assert got[0] == ref[0], graph
        for a, b in zip(got[1:], ref[1:]):
            assert torch.equal(a, b), graph


def _run_gpt2(pg, graph, steps=3, zero=False):
    E, H, S, B, L, V = 768, 12, 128, 2, 2, 1000
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16", zero=zero)
    layers = [nnt_inputs.make_params(E, seed=9, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    shell = nnt_inputs.make_shell_params(V, S, E, seed=10, init="gpt2")
    gm = model.GPT2Model(sc, V, layers, shell, process_group=pg)
    if graph:
        gm.enable_graph()
    losses = []
    for t in range(steps):
        tok = torch.as_tensor(nnt_inputs.make_ids(V, S, 0, B, seed=80 + t)).cuda()
        losses.append(gm.train_step(tok[:, :S].contiguous(), tok[:, 1:].contiguous()).item())
    torch.cuda.synchronize()
    return losses, gm.w.clone(), gm.m.clone(), gm.stack.w.clone(), gm.stack.v.clone()


@pytest.mark.timeout(300)
def test_dp_gpt2_world1_equals_single_gpu_bitwise(pg):
    """The full model's DP path (block buckets + the shell bucket all-reduced on the comm stream,
    Adam per bucket) equals the single-GPU path bitwise, eager and graph-captured."""
    ref = _run_gpt2(None, graph=False)
    for graph in (False, True):
        got = _run_gpt2(pg, graph=graph)
        assert got[0] == ref[0], graph
        for a, b in zip(got[1:], ref[1:]):
            assert torch.equal(a, b), graph


@pytest.mark.timeout(300)
def test_zero1_world1_equals_single_gpu_bitwise(pg):
    """ZeRO-1 (StackConfig.zero) through NCCL: per bucket an in-place
    reduce-scatter, Adam on the owned slice with compact state, an in-place all-gather of the
    fp32 parameters and the bf16 shadow conversion -- block stack and full model, eager and
    graph-captured.  At world size 1 every collective is the identity, so the step must equal
    the single-GPU path bitwise (the ranks>1 bookkeeping is tests/test_dp_host.py's gloo test)."""
    ref = _run(None, graph=False)
    for graph in (False, True):
        got = _run(pg, graph=graph, zero=True)
        assert got[0] == ref[0], graph
        for a, b in zip(got[1:], ref[1:]):
            assert torch.equal(a, b), graph
    ref = _run_gpt2(None, graph=False)
    for graph in (False, True):
        got = _run_gpt2(pg, graph=graph, zero=True)
        assert got[0] == ref[0], graph
        for a, b in zip(got[1:], ref[1:]):
            assert torch.equal(a, b), graph
