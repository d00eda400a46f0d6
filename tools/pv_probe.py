"""PV-shaped batched GEMM (O = P V, causal A_LOWER) timed at several batch counts: separates
DRAM-bound behaviour (time ~ batch) from fixed / issue overheads.  Graph-replayed launches."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_13236_b200 import nnt  # noqa: E402

S, H, Dh = 1024, 12, 64
E = H * Dh
bf = dict(device="cuda", dtype=torch.bfloat16)
for B in (1, 2, 4, 8, 16):
    P = torch.randn(B, H, S, S, **bf) * 0.01
    qkv = torch.randn(B * S, 3 * E, **bf)
    O = torch.empty(B * S, E, **bf)
    epi = nnt.make_epilogue(causal=2)

    def run():
        nnt.nnt_tile_gemm(0, 0, S, Dh, S, (B, H), 1.0, P, 1, S, (H * S * S, S * S), qkv.data_ptr() + 2 * 2 * E, 1,
                          3 * E, (S * 3 * E, Dh), 0.0, O, 1, E, (S * E, Dh), None, epi)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            run()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    pbytes = B * H * 36 * 128 * 128 * 2
    print(f"B={B:3d} {us:8.1f} us  P {pbytes / 1e6:7.1f} MB  {pbytes / us / 1e3:7.0f} GB/s")
