"""Diagnose DP(world 1) vs single-GPU step differences."""
import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import nnt_inputs
from paper_2504_13236_b200 import model

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=torch.device("cuda", 0))
E, H, S, B, L = 768, 12, 256, 2, 2

def run(pg, graph=False, sync=False, steps=3):
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16")
    layers = [nnt_inputs.make_params(E, seed=9, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    st = model.BlockStack(sc, layers, process_group=pg)
    if sync and pg is not None:
        orig = st._reduce_bucket
        def rb(*a):
            torch.cuda.synchronize(); orig(*a); torch.cuda.synchronize()
        st._reduce_bucket = rb
    if graph:
        st.enable_graph()
    out = []
    for t in range(steps):
        x = torch.as_tensor(nnt_inputs.make_x(E, S, 0, B, seed=70 + t)).cuda()
        r = torch.as_tensor(nnt_inputs.make_r(E, S, 0, B, seed=70 + t)).cuda()
        loss = st.train_step(x, r).item()
        torch.cuda.synchronize()
        out.append((loss, st.w.clone(), st.g.clone()))
    return out

ref = run(None)
for name, kw in (("dp", {}), ("dp_sync", {"sync": True}), ("dp_graph", {"graph": True})):
    try:
        got = run(dist.group.WORLD, **kw)
    except Exception as exc:
        print(name, "FAILED", repr(exc)[:300]); continue
    for t, (a, b) in enumerate(zip(got, ref)):
        print(name, t, a[0] == b[0], a[0] - b[0], (a[1] - b[1]).abs().max().item(), (a[2] - b[2]).abs().max().item())
dist.destroy_process_group()
