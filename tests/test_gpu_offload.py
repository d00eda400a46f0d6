"""Optimizer state in pinned host memory (StackConfig.offload, offload.py).

The moments live in host RAM and are streamed through two device staging slots around the
same libnnt update kernel, so parameters, moments and losses must equal the
device-resident run bitwise: block stack and full model, eager and graph-captured, Adam
and SGD, a chunk size that leaves a ragged last chunk, and the DP path (world-size-1 NCCL
group, update per bucket on the communication stream)."""
import socket

import pytest
import torch

import nnt_inputs
from gpu_util import dev

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_13236_b200 import model

E, H, S, B, L, V = 768, 12, 128, 2, 2, 1000


def _stack(offload, graph, optimizer="adam", pg=None, chunk=None, steps=3):
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16", offload=offload, optimizer=optimizer,
                           weight_decay=0.01)
    layers = [nnt_inputs.make_params(E, seed=9, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    st = model.BlockStack(sc, layers, process_group=pg)
    if chunk and offload:
        st.host_state.chunk = chunk
    if graph:
        st.enable_graph()
    losses = []
    for t in range(steps):
        x = dev(nnt_inputs.make_x(E, S, 0, B, seed=70 + t))
        r = dev(nnt_inputs.make_r(E, S, 0, B, seed=70 + t))
        losses.append(st.train_step(x, r).item())
    torch.cuda.synchronize()
    out = [losses, st.w.clone(), st.w16.clone(), st.m.cpu().clone()]
    if optimizer == "adam":
        out.append(st.v.cpu().clone())
    if offload:
        assert st.m.device.type == "cpu" and st.m.is_pinned()
    return out


def _same(a, b):
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        assert torch.equal(x.cpu(), y.cpu())


@pytest.mark.timeout(300)
@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_offload_stack_bitwise(optimizer):
    ref = _stack(False, False, optimizer)
    _same(_stack(True, False, optimizer), ref)
    _same(_stack(True, False, optimizer, chunk=100_003), ref)  # many chunks, ragged tail
    _same(_stack(True, True, optimizer, chunk=1_000_003), ref)


def _gpt2(offload, graph, pg=None, chunk=None, steps=3):
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16", offload=offload)
    layers = [nnt_inputs.make_params(E, seed=9, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    shell = nnt_inputs.make_shell_params(V, S, E, seed=10, init="gpt2")
    gm = model.GPT2Model(sc, V, layers, shell, process_group=pg)
    if chunk and offload:
        gm.host_state.chunk = chunk
        gm.stack.host_state.chunk = chunk
    if graph:
        gm.enable_graph()
    losses = []
    for t in range(steps):
        tok = torch.as_tensor(nnt_inputs.make_ids(V, S, 0, B, seed=80 + t)).cuda()
        losses.append(gm.train_step(tok[:, :S].contiguous(), tok[:, 1:].contiguous()).item())
    torch.cuda.synchronize()
    return [losses, gm.w.clone(), gm.m.cpu().clone(), gm.v.cpu().clone(), gm.stack.w.clone(),
            gm.stack.v.cpu().clone()]


@pytest.mark.timeout(300)
def test_offload_gpt2_bitwise():
    ref = _gpt2(False, False)
    _same(_gpt2(True, False, chunk=300_007), ref)
    _same(_gpt2(True, True), ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_offload_dp_world1_bitwise():
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        ref = _stack(False, False)
        pg = dist.group.WORLD
        _same(_stack(True, False, pg=pg), ref)
        _same(_stack(True, True, pg=pg), ref)
        refg = _gpt2(False, False)
        _same(_gpt2(True, True, pg=pg), refg)
    finally:
        if own:
            dist.destroy_process_group()


# ------------------------------------------------------------------ saved activations in host RAM
def _stack_act(n_off, graph, L_=4, steps=2):
    sc = model.StackConfig(L=L_, E=E, H=H, S=S, B=B, dtype="bf16", act_offload=n_off)
    layers = [nnt_inputs.make_params(E, seed=19, layer=l, init="gpt2", n_layers=L_) for l in range(L_)]
    st = model.BlockStack(sc, layers)
    if n_off:
        assert all(t.device.type == "cpu" and t.is_pinned() for t in st.act_host.host)
        assert len(st.act_host.slots) == min(2, n_off)
    if graph:
        st.enable_graph()
    losses = []
    for t in range(steps):
        x = dev(nnt_inputs.make_x(E, S, 0, B, seed=90 + t))
        r = dev(nnt_inputs.make_r(E, S, 0, B, seed=90 + t))
        losses.append(st.train_step(x, r).item())
    torch.cuda.synchronize()
    return [losses, st.w.clone(), st.w16.clone(), st.m.clone(), st.v.clone()]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n_off", [1, 2, 3, 4])
def test_activation_offload_stack_bitwise(n_off):
    """StackConfig.act_offload (offload.HostActivations): the saved workspaces of
    the lowest n_off of 4 layers go to pinned host RAM after their forward and come back before
    their backward (n_off >= 3 exercises the prefetch into a reused slot).  Bitwise equal to the
    resident run, eager and graph-captured."""
    ref = _stack_act(0, False)
    _same(_stack_act(n_off, False), ref)
    _same(_stack_act(n_off, True), ref)


@pytest.mark.timeout(300)
def test_activation_offload_gpt2_bitwise():
    def run(n_off, graph):
        sc = model.StackConfig(L=3, E=E, H=H, S=S, B=B, dtype="bf16", act_offload=n_off, offload=n_off > 0)
        layers = [nnt_inputs.make_params(E, seed=29, layer=l, init="gpt2", n_layers=3) for l in range(3)]
        shell = nnt_inputs.make_shell_params(V, S, E, seed=30, init="gpt2")
        gm = model.GPT2Model(sc, V, layers, shell)
        if graph:
            gm.enable_graph()
        losses = []
        for t in range(2):
            tok = torch.as_tensor(nnt_inputs.make_ids(V, S, 0, B, seed=95 + t)).cuda()
            losses.append(gm.train_step(tok[:, :S].contiguous(), tok[:, 1:].contiguous()).item())
        torch.cuda.synchronize()
        return [losses, gm.w.clone(), gm.stack.w.clone(), gm.stack.w16.clone()]
    ref = run(0, False)
    _same(run(3, False), ref)
    _same(run(3, True), ref)
