"""cuBLAS (torch.matmul) timing of the GPT-2 block's projection GEMM shapes: a library reference
point for tools/gemm_bench.py (not on the product path)."""
import sys
import torch

T, E = 8192, int(sys.argv[1]) if len(sys.argv) > 1 else 768
F = 4 * E
bf = dict(device="cuda", dtype=torch.bfloat16)
cases = {"qkv": (T, 3 * E, E), "out": (T, E, E), "fc": (T, F, E), "proj": (T, E, F), "fc_dx": (T, E, F),
         "qkv_dx": (T, E, 3 * E), "proj_dw": (E, F, T), "fc_dw": (F, E, T), "out_dw": (E, E, T),
         "qkv_dw": (3 * E, E, T), "square8192": (8192, 8192, 8192)}
for name, (M, N, K) in cases.items():
    a = torch.randn(M, K, **bf)
    b = torch.randn(K, N, **bf)
    for outdt in (torch.bfloat16, torch.float32):
        if outdt == torch.float32:
            f = lambda: torch.matmul(a, b, out_dtype=torch.float32) if hasattr(torch, "matmul") else None
            try:
                f()
            except Exception:
                continue
        else:
            f = lambda: torch.matmul(a, b)
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        print(f"{name:10s} {str(outdt)[6:]:9s} {M:6d} {N:6d} {K:6d} {us:8.1f} us {2 * M * N * K / us / 1e6:8.1f} TFLOP/s")
