"""One 128 x N output tile with a long K (a single CTA's pipeline, latency-bound): time vs K gives
the per-K-block cost of the TMA -> MMA -> commit loop.  Graph-replayed launches."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_13236_b200 import nnt  # noqa: E402

bf = dict(device="cuda", dtype=torch.bfloat16)
for N in (64, 256):
    for K in (256, 1024, 4096, 16384):
        A = torch.randn(128, K, **bf)
        B = torch.randn(N, K, **bf)
        C = torch.empty(128, N, **bf)

        def run():
            nnt.nnt_tile_gemm(0, 1, 128, N, K, None, 1.0, A, 1, K, None, B, 1, K, None, 0.0, C, 1, N, None)
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                run()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 100
        print(f"N={N:4d} K={K:6d} {us:8.2f} us  {us * 1e3 / (K / 64):7.1f} ns per K-block")
