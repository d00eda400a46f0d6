"""Times the three tied-LM-head GEMMs of GPT-2 (logits = h wte^T, dh = dlogits wte, dwte =
dlogits^T h) through nnt_tile_gemm, graph-replayed.   python tools/lmhead_bench.py [E]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_13236_b200 import nnt  # noqa: E402

T, V = 8192, 50257
E = int(sys.argv[1]) if len(sys.argv) > 1 else 768
Vp = -(-V // 8) * 8
bf = dict(device="cuda", dtype=torch.bfloat16)
h = torch.randn(T, E, **bf)
w = torch.randn(V, E, **bf) * 0.02
lg = torch.randn(T, Vp, **bf) * 0.01
dh = torch.empty(T, E, device="cuda")
dw = torch.empty(V, E, device="cuda")
wsb = nnt.nnt_tile_gemm_workspace_bytes(T, E, V, nnt.NNT_F32)
ws = torch.empty(max(wsb, 16), device="cuda", dtype=torch.uint8)
epi = nnt.make_epilogue(workspace=ws) if wsb else None
cases = {
    "logits": lambda: nnt.nnt_tile_gemm(0, 1, T, V, E, None, 1.0, h, 1, E, None, w, 1, E, None, 0.0, lg, 1, Vp, None),
    "dh": lambda: nnt.nnt_tile_gemm(0, 0, T, E, V, None, 1.0, lg, 1, Vp, None, w, 1, E, None, 0.0, dh, 0, E, None,
                                    None, epi),
    "dwte": lambda: nnt.nnt_tile_gemm(1, 0, V, E, T, None, 1.0, lg, 1, Vp, None, h, 1, E, None, 0.0, dw, 0, E, None),
}
for name, fn in cases.items():
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(5):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"{name:8s} {us:8.1f} us  {2 * T * V * E / us / 1e6:8.1f} TFLOP/s")
a, b = h, w
for _ in range(3):
    torch.matmul(a, b.t())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    torch.matmul(a, b.t())
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 10
print(f"cuBLAS logits {us:8.1f} us  {2 * T * V * E / us / 1e6:8.1f} TFLOP/s")
